"""UNet ε-prediction (ORACLE — test infrastructure only).

What one row of the step-level batch computes:
ε = UNet(c_in·x_r, t_r, ctx_r). Rows are independent (I1), so the batch is just a
loop-free stack of rows. Structure follows diffusers UNet2DConditionModel (R1).
"""
from __future__ import annotations

import numpy as np

from . import nn
from .configs import UNetConfig, unet_structure


def resnet(P, p, x, temb, groups, eps):
    """ResnetBlock2D: GN→SiLU→conv1 (+ Linear(SiLU(temb))) → GN→SiLU→conv2, + shortcut."""
    h = nn.silu(nn.group_norm(x, groups, P[p + ".norm1.weight"], P[p + ".norm1.bias"], eps))
    h = nn.conv2d(h, P[p + ".conv1.weight"], P[p + ".conv1.bias"])
    if temb is not None:
        tp = nn.linear(nn.silu(temb), P[p + ".time_emb_proj.weight"], P[p + ".time_emb_proj.bias"])
        h = h + tp[:, :, None, None]
    h = nn.silu(nn.group_norm(h, groups, P[p + ".norm2.weight"], P[p + ".norm2.bias"], eps))
    h = nn.conv2d(h, P[p + ".conv2.weight"], P[p + ".conv2.bias"])
    if (p + ".conv_shortcut.weight") in P:
        x = nn.conv2d(x, P[p + ".conv_shortcut.weight"], P[p + ".conv_shortcut.bias"], pad=0)
    return x + h


def _mha(q, k, v, heads):
    """[N, L, C] → split heads → attention → merge."""
    N, L, C = q.shape
    S = k.shape[1]
    d = C // heads
    qh = q.reshape(N, L, heads, d).transpose(0, 2, 1, 3)
    kh = k.reshape(N, S, heads, d).transpose(0, 2, 1, 3)
    vh = v.reshape(N, S, heads, d).transpose(0, 2, 1, 3)
    o = nn.attention(qh, kh, vh)
    return o.transpose(0, 2, 1, 3).reshape(N, L, C)


def transformer(P, p, x, ctx, cfg: UNetConfig):
    """Transformer2DModel (conv proj_in/out) with one BasicTransformerBlock (App. C)."""
    N, C, H, W = x.shape
    res = x
    h = nn.group_norm(x, cfg.groups, P[p + ".norm.weight"], P[p + ".norm.bias"], cfg.eps_tf_gn)
    h = nn.conv2d(h, P[p + ".proj_in.weight"], P[p + ".proj_in.bias"], pad=0)
    h = h.reshape(N, C, H * W).transpose(0, 2, 1)              # [N, L, C]
    b = p + ".transformer_blocks.0"
    n1 = nn.layer_norm(h, P[b + ".norm1.weight"], P[b + ".norm1.bias"], cfg.eps_ln)
    q = nn.linear(n1, P[b + ".attn1.to_q.weight"])
    k = nn.linear(n1, P[b + ".attn1.to_k.weight"])
    v = nn.linear(n1, P[b + ".attn1.to_v.weight"])
    h = h + nn.linear(_mha(q, k, v, cfg.heads), P[b + ".attn1.to_out.0.weight"], P[b + ".attn1.to_out.0.bias"])
    n2 = nn.layer_norm(h, P[b + ".norm2.weight"], P[b + ".norm2.bias"], cfg.eps_ln)
    q = nn.linear(n2, P[b + ".attn2.to_q.weight"])
    k = nn.linear(ctx, P[b + ".attn2.to_k.weight"])
    v = nn.linear(ctx, P[b + ".attn2.to_v.weight"])
    h = h + nn.linear(_mha(q, k, v, cfg.heads), P[b + ".attn2.to_out.0.weight"], P[b + ".attn2.to_out.0.bias"])
    n3 = nn.layer_norm(h, P[b + ".norm3.weight"], P[b + ".norm3.bias"], cfg.eps_ln)
    pr = nn.linear(n3, P[b + ".ff.net.0.proj.weight"], P[b + ".ff.net.0.proj.bias"])
    hh, gate = np.split(pr, 2, axis=-1)                          # diffusers order (R30)
    h = h + nn.linear(hh * nn.gelu(gate), P[b + ".ff.net.2.weight"], P[b + ".ff.net.2.bias"])
    h = h.transpose(0, 2, 1).reshape(N, C, H, W)
    h = nn.conv2d(h, P[p + ".proj_out.weight"], P[p + ".proj_out.bias"], pad=0)
    return h + res


def time_embedding(P, cfg: UNetConfig, t, dtype):
    e = nn.timestep_embedding(t, cfg.block_out[0], dtype)
    e = nn.linear(e, P["time_embedding.linear_1.weight"], P["time_embedding.linear_1.bias"])
    e = nn.silu(e)
    return nn.linear(e, P["time_embedding.linear_2.weight"], P["time_embedding.linear_2.bias"])


def forward(P, cfg: UNetConfig, x, t, ctx):
    """ε = UNet(x, t, ctx).  x [N,4,H,W], t [N] (integer timesteps), ctx [N, L, D]."""
    dtype = x.dtype
    temb = time_embedding(P, cfg, t, dtype)
    down, up = unet_structure(cfg)
    eps = cfg.eps_resnet
    h = nn.conv2d(x, P["conv_in.weight"], P["conv_in.bias"])
    skips = [h]
    for i, blk in enumerate(down):
        for j in range(len(blk["res"])):
            h = resnet(P, f"down_blocks.{i}.resnets.{j}", h, temb, cfg.groups, eps)
            if blk["attn"]:
                h = transformer(P, f"down_blocks.{i}.attentions.{j}", h, ctx, cfg)
            skips.append(h)
        if blk["down"]:
            h = nn.conv2d(h, P[f"down_blocks.{i}.downsamplers.0.conv.weight"],
                          P[f"down_blocks.{i}.downsamplers.0.conv.bias"], stride=2, pad=1)
            skips.append(h)
    h = resnet(P, "mid_block.resnets.0", h, temb, cfg.groups, eps)
    h = transformer(P, "mid_block.attentions.0", h, ctx, cfg)
    h = resnet(P, "mid_block.resnets.1", h, temb, cfg.groups, eps)
    for i, blk in enumerate(up):
        for j in range(len(blk["res"])):
            s = skips.pop()
            h = np.concatenate([h, s], axis=1)                  # cat([h, skip]) (App. C)
            h = resnet(P, f"up_blocks.{i}.resnets.{j}", h, temb, cfg.groups, eps)
            if blk["attn"]:
                h = transformer(P, f"up_blocks.{i}.attentions.{j}", h, ctx, cfg)
        if blk["up"]:
            h = nn.upsample_nearest2x(h)
            h = nn.conv2d(h, P[f"up_blocks.{i}.upsamplers.0.conv.weight"], P[f"up_blocks.{i}.upsamplers.0.conv.bias"])
    assert not skips
    h = nn.silu(nn.group_norm(h, cfg.groups, P["conv_norm_out.weight"], P["conv_norm_out.bias"], eps))
    return nn.conv2d(h, P["conv_out.weight"], P["conv_out.bias"])

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


def _proj(P, name, h_tokens, cfg):
    """proj_in / proj_out on token-major [N, L, C]: a 1×1 conv (SD-1.5) or a Linear (SDXL) — the
    same contraction, weights [C][C](1×1)."""
    w = P[name + ".weight"]
    return nn.linear(h_tokens, w.reshape(w.shape[0], w.shape[1]), P[name + ".bias"])


def basic_block(P, b, h, ctx, cfg: UNetConfig, heads):
    """BasicTransformerBlock: LN→self-attn→+, LN→cross-attn→+, LN→GEGLU FF→+ (App. C)."""
    n1 = nn.layer_norm(h, P[b + ".norm1.weight"], P[b + ".norm1.bias"], cfg.eps_ln)
    q = nn.linear(n1, P[b + ".attn1.to_q.weight"])
    k = nn.linear(n1, P[b + ".attn1.to_k.weight"])
    v = nn.linear(n1, P[b + ".attn1.to_v.weight"])
    h = h + nn.linear(_mha(q, k, v, heads), P[b + ".attn1.to_out.0.weight"], P[b + ".attn1.to_out.0.bias"])
    n2 = nn.layer_norm(h, P[b + ".norm2.weight"], P[b + ".norm2.bias"], cfg.eps_ln)
    q = nn.linear(n2, P[b + ".attn2.to_q.weight"])
    k = nn.linear(ctx, P[b + ".attn2.to_k.weight"])
    v = nn.linear(ctx, P[b + ".attn2.to_v.weight"])
    h = h + nn.linear(_mha(q, k, v, heads), P[b + ".attn2.to_out.0.weight"], P[b + ".attn2.to_out.0.bias"])
    n3 = nn.layer_norm(h, P[b + ".norm3.weight"], P[b + ".norm3.bias"], cfg.eps_ln)
    pr = nn.linear(n3, P[b + ".ff.net.0.proj.weight"], P[b + ".ff.net.0.proj.bias"])
    hh, gate = np.split(pr, 2, axis=-1)                          # diffusers order (R30)
    return h + nn.linear(hh * nn.gelu(gate), P[b + ".ff.net.2.weight"], P[b + ".ff.net.2.bias"])


def transformer(P, p, x, ctx, cfg: UNetConfig, depth=1):
    """Transformer2DModel: GN → proj_in → `depth` BasicTransformerBlocks → proj_out → + x (App. C)."""
    N, C, H, W = x.shape
    res = x
    h = nn.group_norm(x, cfg.groups, P[p + ".norm.weight"], P[p + ".norm.bias"], cfg.eps_tf_gn)
    h = h.reshape(N, C, H * W).transpose(0, 2, 1)              # [N, L, C]
    h = _proj(P, p + ".proj_in", h, cfg)
    for d in range(depth):
        h = basic_block(P, p + f".transformer_blocks.{d}", h, ctx, cfg, cfg.heads_at(C))
    h = _proj(P, p + ".proj_out", h, cfg)
    return h.transpose(0, 2, 1).reshape(N, C, H, W) + res


def time_embedding(P, cfg: UNetConfig, t, dtype):
    e = nn.timestep_embedding(t, cfg.block_out[0], dtype)
    e = nn.linear(e, P["time_embedding.linear_1.weight"], P["time_embedding.linear_1.bias"])
    e = nn.silu(e)
    return nn.linear(e, P["time_embedding.linear_2.weight"], P["time_embedding.linear_2.bias"])


def added_embedding(P, cfg: UNetConfig, pooled, time_ids, dtype):
    """SDXL "text_time" added conditioning (R27): sinusoid(time_id, add_time_dim) for each of the 6
    ids, flattened, ‖ pooled text embedding → add_embedding MLP (Linear → SiLU → Linear)."""
    N = pooled.shape[0]
    tid = np.asarray(time_ids).reshape(N * 6)
    te = nn.timestep_embedding(tid, cfg.add_time_dim, dtype).reshape(N, 6 * cfg.add_time_dim)
    a = np.concatenate([te, pooled.astype(dtype)], axis=1)
    a = nn.linear(a, P["add_embedding.linear_1.weight"], P["add_embedding.linear_1.bias"])
    a = nn.silu(a)
    return nn.linear(a, P["add_embedding.linear_2.weight"], P["add_embedding.linear_2.bias"])


def forward(P, cfg: UNetConfig, x, t, ctx, pooled=None, time_ids=None):
    """ε = UNet(x, t, ctx).  x [N,4,H,W], t [N] (integer timesteps), ctx [N, L, D]; SDXL also
    pooled [N, pooled_dim] and time_ids [N, 6] (default R27's (1024,1024,0,0,1024,1024))."""
    dtype = x.dtype
    temb = time_embedding(P, cfg, t, dtype)
    if cfg.add_time_dim:
        if time_ids is None:
            from .configs import SDXL_TIME_IDS
            time_ids = np.tile(np.array(SDXL_TIME_IDS, dtype=np.float64), (x.shape[0], 1))
        temb = temb + added_embedding(P, cfg, pooled, time_ids, dtype)
    down, up = unet_structure(cfg)
    L = len(cfg.block_out)
    eps = cfg.eps_resnet
    h = nn.conv2d(x, P["conv_in.weight"], P["conv_in.bias"])
    skips = [h]
    for i, blk in enumerate(down):
        for j in range(len(blk["res"])):
            h = resnet(P, f"down_blocks.{i}.resnets.{j}", h, temb, cfg.groups, eps)
            if blk["attn"]:
                h = transformer(P, f"down_blocks.{i}.attentions.{j}", h, ctx, cfg, cfg.depth(i))
            skips.append(h)
        if blk["down"]:
            h = nn.conv2d(h, P[f"down_blocks.{i}.downsamplers.0.conv.weight"],
                          P[f"down_blocks.{i}.downsamplers.0.conv.bias"], stride=2, pad=1)
            skips.append(h)
    h = resnet(P, "mid_block.resnets.0", h, temb, cfg.groups, eps)
    h = transformer(P, "mid_block.attentions.0", h, ctx, cfg, cfg.mid_depth)
    h = resnet(P, "mid_block.resnets.1", h, temb, cfg.groups, eps)
    for i, blk in enumerate(up):
        for j in range(len(blk["res"])):
            s = skips.pop()
            h = np.concatenate([h, s], axis=1)                  # cat([h, skip]) (App. C)
            h = resnet(P, f"up_blocks.{i}.resnets.{j}", h, temb, cfg.groups, eps)
            if blk["attn"]:
                h = transformer(P, f"up_blocks.{i}.attentions.{j}", h, ctx, cfg, cfg.depth(L - 1 - i))
        if blk["up"]:
            h = nn.upsample_nearest2x(h)
            h = nn.conv2d(h, P[f"up_blocks.{i}.upsamplers.0.conv.weight"], P[f"up_blocks.{i}.upsamplers.0.conv.bias"])
    assert not skips
    h = nn.silu(nn.group_norm(h, cfg.groups, P["conv_norm_out.weight"], P["conv_norm_out.bias"], eps))
    return nn.conv2d(h, P["conv_out.weight"], P["conv_out.bias"])

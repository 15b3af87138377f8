"""Experiment (not a test): which bf16 STORAGE sites of the GPU path carry the error? A GPU-faithful
emulation: every conv / linear operand is rounded to bf16 (the tensor cores read bf16), the attention
probabilities P are rounded (P·V in bf16), and each stored tensor is rounded only if its site is in
`sites`:
  h1     conv1 output (+temb)            → GroupNorm 2 input
  sc     1×1 shortcut output             → residual of conv2
  res    conv2 + residual                → resblock output (residual stream, skips, next GN input)
  tfh    transformer-internal residual stream (proj_in out, attn / xattn out-proj + h, FF2 + h)
  tfo    proj_out + x                    → transformer output (residual stream)
  io     conv_in / downsampler / upsampler conv outputs
Usage: python tests/experiments/bf16_sites.py [sd15|tiny] [latent] [n_steps]"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])
import synth  # noqa: E402
from oracle import configs, nn, pipeline, unet, vae  # noqa: E402

q = synth.bf16_round
ALL = ("h1", "sc", "res", "tfh", "tfo", "io")
S = set()
_conv, _lin, _soft = nn.conv2d, nn.linear, nn.softmax
_res, _tf, _bb = unet.resnet, unet.transformer, unet.basic_block


def st(x, site):
    return q(x) if site in S else x


def conv(x, w, b=None, stride=1, pad=None):
    return _conv(q(x), w, b, stride, pad)


def lin(x, w, b=None):
    return _lin(q(x), w, b)


def resnet(P, p, x, temb, groups, eps):
    h = nn.silu(nn.group_norm(x, groups, P[p + ".norm1.weight"], P[p + ".norm1.bias"], eps))
    h = conv(h, P[p + ".conv1.weight"], P[p + ".conv1.bias"])
    if temb is not None:
        tp = lin(nn.silu(temb), P[p + ".time_emb_proj.weight"], P[p + ".time_emb_proj.bias"])
        h = h + tp[:, :, None, None]
    h = st(h, "h1")
    h = nn.silu(nn.group_norm(h, groups, P[p + ".norm2.weight"], P[p + ".norm2.bias"], eps))
    h = conv(h, P[p + ".conv2.weight"], P[p + ".conv2.bias"])
    if (p + ".conv_shortcut.weight") in P:
        x = st(conv(x, P[p + ".conv_shortcut.weight"], P[p + ".conv_shortcut.bias"], pad=0), "sc")
    return st(x + h, "res")


def basic_block(P, b, h, ctx, cfg, heads):
    n1 = nn.layer_norm(h, P[b + ".norm1.weight"], P[b + ".norm1.bias"], cfg.eps_ln)
    qq, k, v = (lin(n1, P[b + f".attn1.to_{t}.weight"]) for t in "qkv")
    h = st(h + lin(unet._mha(q(qq), q(k), q(v), heads), P[b + ".attn1.to_out.0.weight"],
                   P[b + ".attn1.to_out.0.bias"]), "tfh")
    n2 = nn.layer_norm(h, P[b + ".norm2.weight"], P[b + ".norm2.bias"], cfg.eps_ln)
    qq = lin(n2, P[b + ".attn2.to_q.weight"])
    k = lin(ctx, P[b + ".attn2.to_k.weight"])
    v = lin(ctx, P[b + ".attn2.to_v.weight"])
    h = st(h + lin(unet._mha(q(qq), q(k), q(v), heads), P[b + ".attn2.to_out.0.weight"],
                   P[b + ".attn2.to_out.0.bias"]), "tfh")
    n3 = nn.layer_norm(h, P[b + ".norm3.weight"], P[b + ".norm3.bias"], cfg.eps_ln)
    pr = lin(n3, P[b + ".ff.net.0.proj.weight"], P[b + ".ff.net.0.proj.bias"])
    hh, gate = np.split(pr, 2, axis=-1)
    return st(h + lin(hh * nn.gelu(gate), P[b + ".ff.net.2.weight"], P[b + ".ff.net.2.bias"]), "tfh")


def transformer(P, p, x, ctx, cfg, depth=1):
    N, C, H, W = x.shape
    h = nn.group_norm(x, cfg.groups, P[p + ".norm.weight"], P[p + ".norm.bias"], cfg.eps_tf_gn)
    h = h.reshape(N, C, H * W).transpose(0, 2, 1)
    w = P[p + ".proj_in.weight"]
    h = st(lin(h, w.reshape(w.shape[0], w.shape[1]), P[p + ".proj_in.bias"]), "tfh")
    for d in range(depth):
        h = basic_block(P, p + f".transformer_blocks.{d}", h, ctx, cfg, cfg.heads_at(C))
    w = P[p + ".proj_out.weight"]
    h = lin(h, w.reshape(w.shape[0], w.shape[1]), P[p + ".proj_out.bias"])
    return st(h.transpose(0, 2, 1).reshape(N, C, H, W) + x, "tfo")


def install(sites):
    S.clear()
    S.update(sites)
    nn.conv2d = lambda *a, **k: st(conv(*a, **k), "io")     # the convs forward() / vae call directly
    nn.linear = lin
    nn.softmax = lambda s, axis=-1: q(_soft(s, axis))
    unet.resnet, unet.transformer, unet.basic_block = resnet, transformer, basic_block
    vae._resnet = resnet


def uninstall():
    nn.conv2d, nn.linear, nn.softmax = _conv, _lin, _soft
    unet.resnet, unet.transformer, unet.basic_block = _res, _tf, _bb
    vae._resnet = _res


def rel(a, b):
    return float(np.linalg.norm((a - b).astype(np.float64)) / np.linalg.norm(b.astype(np.float64)))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    hw = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    cfg = {"sd15": configs.SD15_UNET, "tiny": configs.TINY_UNET}[name]
    vc = {"sd15": configs.SD_VAE, "tiny": configs.TINY_VAE}[name]
    L, D = (77, 768) if name == "sd15" else (8, 32)
    P = configs.unet_params(cfg, 0, np.float32, bf16_weights=True)
    V = configs.vae_params(vc, 0, np.float32, bf16_weights=True)
    cu = q(synth.uncond_embedding(0, L, D))
    emb, xT = q(synth.text_embedding(5, 0, L, D)), synth.initial_noise(5, 0, hw, hw)
    ref = pipeline.denoise(P, cfg, xT, emb, cu, n, 7.5, "ddim")
    ref_img = vae.decode(V, vc, ref[None])
    variants = [ALL, ()] + [tuple(s for s in ALL if s != x) for x in ALL] + [(x,) for x in ALL]
    for sites in variants:
        install(sites)
        try:
            x = pipeline.denoise(P, cfg, xT, emb, cu, n, 7.5, "ddim")
            img = vae.decode(V, vc, x[None])
            img_l = vae.decode(V, vc, ref[None])
        finally:
            uninstall()
        print(f"{name} {hw} n={n} stored bf16: {'+'.join(sites) or '(none)':24s} latent {rel(x, ref):.3e}  "
              f"image {rel(img, ref_img):.3e}  vae-only {rel(img_l, ref_img):.3e}", flush=True)


if __name__ == "__main__":
    main()

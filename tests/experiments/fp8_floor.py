"""Experiment (not a test): SURVEY §8(f) rank 3's FP8 accuracy study, before any kind::f8f6f4 kernel.
The oracle runs with the tensor-core OPERANDS of every conv / linear rounded to FP8 (E4M3, per-tensor
scale = amax / 448, round-to-nearest-even on the 3-bit mantissa) — weights and activations both — while
storage stays fp32 (the most favourable case), and reports final-latent / image rel-L2 against the plain
fp32 oracle, next to the same run with fp16 and bf16 operands (what the GPU modes use).

  python tests/experiments/fp8_floor.py [tiny|sd15] [latent] [n_steps]"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])
import synth  # noqa: E402
from oracle import configs, nn, pipeline, vae  # noqa: E402

_conv, _lin = nn.conv2d, nn.linear


def e4m3(x):
    """Round to FP8 E4M3 with a per-tensor scale (amax → 448): 3 mantissa bits, min normal 2^-6 (scaled)."""
    x = np.asarray(x, np.float32)
    amax = float(np.abs(x).max())
    if amax == 0:
        return x
    s = 448.0 / amax
    y = x * s
    a = np.abs(y)
    e = np.floor(np.log2(np.maximum(a, 2.0 ** -9)))
    e = np.maximum(e, -6.0)                       # subnormals below 2^-6: fixed spacing 2^-9
    q = 2.0 ** (e - 3)                            # 3 mantissa bits
    r = np.round(a / q) * q                       # numpy rounds half to even
    return (np.sign(y) * np.minimum(r, 448.0) / s).astype(np.float32)


def f16(x):
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float32)


def install(rnd):
    nn.conv2d = lambda x, w, b=None, stride=1, pad=None: _conv(rnd(x), rnd(w), b, stride, pad)
    nn.linear = lambda x, w, b=None: _lin(rnd(x), rnd(w), b)


def uninstall():
    nn.conv2d, nn.linear = _conv, _lin


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
    cu = synth.bf16_round(synth.uncond_embedding(0, L, D))
    emb = synth.bf16_round(synth.text_embedding(5, 0, L, D))
    xT = synth.initial_noise(5, 0, hw, hw)
    ref = pipeline.denoise(P, cfg, xT, emb, cu, n, 7.5, "ddim")
    ref_img = vae.decode(V, vc, ref[None])
    for label, rnd in (("fp16 operands", f16), ("bf16 operands", synth.bf16_round), ("fp8 e4m3 operands", e4m3)):
        install(rnd)
        try:
            x = pipeline.denoise(P, cfg, xT, emb, cu, n, 7.5, "ddim")
            img = vae.decode(V, vc, x[None])
            img_vae_only = vae.decode(V, vc, ref[None])
        finally:
            uninstall()
        print(f"{name} {hw}² n={n} {label:18s}: latent {rel(x, ref):.3e}  image {rel(img, ref_img):.3e}  "
              f"VAE alone {rel(img_vae_only, ref_img):.3e}", flush=True)


if __name__ == "__main__":
    main()

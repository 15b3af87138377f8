"""Experiment (not a test): where does the bf16 path's ε error come from? Runs the oracle UNet with
bf16 rounding emulated at chosen sites and reports single-step ε rel-L2 vs the plain fp32 oracle,
for ε_c, ε_u and the CFG combine ε̃ (g = 7.5).

Sites: "op"  = every conv / linear operand (GN, LN, attention output … as the tensor cores read them)
       "out" = every conv / linear output stored in bf16 (incl. the fused residual sums)
       "p"   = attention probabilities P rounded before P·V
Usage: python tests/experiments/bf16_floor.py [latent_hw] [model]"""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])
import synth  # noqa: E402
from oracle import configs, nn, sampling, unet  # noqa: E402

q = synth.bf16_round
orig = {k: getattr(nn, k) for k in ("conv2d", "linear", "softmax")}
orig_resnet, orig_tf, orig_bb = unet.resnet, unet.transformer, unet.basic_block


def install(sites):
    def conv2d(x, w, b=None, stride=1, pad=None):
        y = orig["conv2d"](q(x) if "op" in sites else x, w, b, stride, pad)
        return q(y) if "out" in sites and "res_f32" not in sites else y

    def linear(x, w, b=None):
        y = orig["linear"](q(x) if "op" in sites else x, w, b)
        return q(y) if "out" in sites and "res_f32" not in sites else y

    def softmax(s, axis=-1):
        p = orig["softmax"](s, axis)
        return q(p) if "p" in sites else p

    nn.conv2d, nn.linear, nn.softmax = conv2d, linear, softmax

    def resnet(*a, **k):
        y = orig_resnet(*a, **k)
        return q(y) if "out" in sites and "res_f32" not in sites else y
    unet.resnet = resnet


def uninstall():
    nn.conv2d, nn.linear, nn.softmax = orig["conv2d"], orig["linear"], orig["softmax"]
    unet.resnet = orig_resnet


def rel(a, b):
    return float(np.linalg.norm((a - b).astype(np.float64)) / np.linalg.norm(b.astype(np.float64)))


def main():
    hw = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    name = sys.argv[2] if len(sys.argv) > 2 else "sd15"
    cfg = {"sd15": configs.SD15_UNET, "tiny": configs.TINY_UNET}[name]
    P = configs.unet_params(cfg, 0, np.float32, bf16_weights=True)
    L, D = (77, 768) if name == "sd15" else (8, 32)
    ctx = q(synth.text_embedding(1, 0, L, D))
    cu = q(synth.uncond_embedding(0, L, D))
    x = synth.initial_noise(1, 0, hw, hw)
    t = int(sampling.timesteps(50)[0])
    X, T, Cx = np.stack([x, x]), np.array([t, t]), np.stack([ctx, cu])
    t0 = time.time()
    ref = unet.forward(P, cfg, X, T, Cx)
    g = np.float32(7.5)
    et_ref = ref[1] + g * (ref[0] - ref[1])
    print(f"{name} latent {hw}: reference {time.time() - t0:.1f} s; |eps_c-eps_u|/|eps_u| = {rel(ref[0], ref[1]):.3e}")
    for sites in (["op"], ["op", "p"], ["op", "out"], ["op", "out", "p"], ["op", "out", "p", "res_f32"], ["out"]):
        install(set(sites))
        try:
            e = unet.forward(P, cfg, X, T, Cx)
        finally:
            uninstall()
        et = e[1] + g * (e[0] - e[1])
        print(f"  sites {'+'.join(sites):22s}: eps_c {rel(e[0], ref[0]):.3e}  eps_u {rel(e[1], ref[1]):.3e}  "
              f"eps~ {rel(et, et_ref):.3e}", flush=True)




def multistep(hw=16, n=4, skip=(2,), name="sd15"):
    """Final-latent (and decoded-image) rel-L2 of a whole n-step DDIM request (g = 7.5, one Skip-CFG
    step) per site set."""
    from oracle import pipeline, vae
    cfg = {"sd15": configs.SD15_UNET, "tiny": configs.TINY_UNET}[name]
    vc = {"sd15": configs.SD_VAE, "tiny": configs.TINY_VAE}[name]
    L, D = (77, 768) if name == "sd15" else (8, 32)
    P = configs.unet_params(cfg, 0, np.float32, bf16_weights=True)
    V = configs.vae_params(vc, 0, np.float32, bf16_weights=True)
    ctx = q(synth.text_embedding(41, 0, L, D))
    cu = q(synth.uncond_embedding(0, L, D))
    xT = synth.initial_noise(41, 0, hw, hw)
    ref = pipeline.denoise(P, cfg, xT, ctx, cu, n, 7.5, "ddim", skip=set(skip))
    ref_img = vae.decode(V, vc, ref[None])
    orig_vr = vae._resnet
    for sites in (["op", "out", "p"], ["op", "p"], ["out"]):
        install(set(sites))

        def vr(*a, **k):
            y = orig_vr(*a, **k)
            return q(y) if "out" in sites else y
        vae._resnet = vr
        try:
            x = pipeline.denoise(P, cfg, xT, ctx, cu, n, 7.5, "ddim", skip=set(skip))
            img = vae.decode(V, vc, x[None])
        finally:
            uninstall()
            vae._resnet = orig_vr
        print(f"  {name} n={n} skip={skip} sites {'+'.join(sites):14s}: final latent rel-L2 {rel(x, ref):.3e}, "
              f"image {rel(img, ref_img):.3e}", flush=True)


def vae_floor(hw=32):
    """VAE decode rel-L2 per site set (the VAE resnets come from oracle.vae._resnet)."""
    from oracle import vae
    V = configs.vae_params(configs.SD_VAE, 0, np.float32, bf16_weights=True)
    z = synth.initial_noise(3, 0, hw, hw)[None]
    ref = vae.decode(V, configs.SD_VAE, z)
    orig_vr = vae._resnet
    for sites in (["op", "out", "p"], ["op", "p"], ["op"], ["out"]):
        install(set(sites))

        def vr(*a, **k):
            y = orig_vr(*a, **k)
            return q(y) if "out" in sites else y
        vae._resnet = vr
        try:
            img = vae.decode(V, configs.SD_VAE, z)
        finally:
            uninstall()
            vae._resnet = orig_vr
        print(f"  VAE latent {hw} sites {'+'.join(sites):14s}: image rel-L2 {rel(img, ref):.3e}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "vae":
        vae_floor(int(sys.argv[2]) if len(sys.argv) > 2 else 32)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "multi":
        multistep(int(sys.argv[2]) if len(sys.argv) > 2 else 16, int(sys.argv[3]) if len(sys.argv) > 3 else 4,
                  name=sys.argv[4] if len(sys.argv) > 4 else "sd15")
    else:
        main()

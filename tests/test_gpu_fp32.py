"""fp32 parity mode (SD_PREC_FP32) against the NumPy oracle: rel-L2 ≤ 1e-4 (north star; SURVEY §8(c)
tolerances, R19 "fp32 mode: everything fp32").

The engine runs the same UNet / VAE graph as the bf16 product path with fp32 weights and activations
on the SIMT fp32 kernels (csrc/fp32.cu). The oracle runs in fp32 with the UNROUNDED fp32 weights and
text embeddings (bf16_weights=False), so the only differences left are summation order and the
transcendental implementations — ~1e-6 per op, far inside 1e-4."""
import numpy as np
import pytest
import torch

import synth
from oracle import configs, pipeline, sampling, unet, vae

pytestmark = pytest.mark.gpu

from paper_2605_08835_b200.engine import Engine  # noqa: E402

TOL32 = 1e-4
U32 = 2.0 ** -24  # fp32 unit roundoff


def eps_part_bound(kappa, x_term, eps_part):
    """Allowed rel-L2 of the ε-part x_new − A·x: TOL32·κ for the kernels, plus the fp32 rounding of the
    A·x term in the GPU's and the oracle's own update (a few ulps of ‖A·x‖), which dominates when the
    ε-part is ~1 % of x (the last DDIM step: A ≈ 1, b ≈ −0.012)."""
    return TOL32 * kappa + 16 * U32 * float(np.linalg.norm(x_term)) / max(float(np.linalg.norm(eps_part)), 1e-30)


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def tiny32():
    eng = Engine("tiny", max_latent_hw=16, b_max=4, precision="fp32")
    ctx_u = synth.uncond_embedding(0, 8, 32)
    eng.set_uncond(torch.from_numpy(ctx_u))
    P = configs.unet_params(configs.TINY_UNET, 0, np.float32)
    V = configs.vae_params(configs.TINY_VAE, 0, np.float32)
    yield eng, P, V, ctx_u
    eng.close()


@pytest.mark.parametrize("sampler", ["ddim", "euler"])
def test_fp32_tiny_four_steps(sampler):
    """CFG#1 in the fp32 mode: 2 requests × 4 steps with CFG on / Skip-CFG mixes, free-running (the
    GPU and the oracle each feed back their own latents); final latents ≤ 1e-4, and every step's
    teacher-forced ε-part ≤ 1e-4·κ (κ = CFG error-propagation factor)."""
    eng = Engine("tiny", max_latent_hw=16, b_max=4, sampler=sampler, precision="fp32")
    try:
        cfg = configs.TINY_UNET
        P = configs.unet_params(cfg, 0, np.float32)
        ctx_u = synth.uncond_embedding(0, 8, 32)
        eng.set_uncond(torch.from_numpy(ctx_u))
        g = [7.5, 5.0]
        ctx = [synth.text_embedding(1, i, 8, 32) for i in range(2)]
        slots = [eng.register(torch.from_numpy(c)) for c in ctx]
        sig = sampling.init_sigma(sampler, 4)
        x0 = [synth.initial_noise(1, i, 8, 8) * np.float32(sig) for i in range(2)]
        lat = [torch.from_numpy(x).cuda() for x in x0]
        xo = [x.copy() for x in x0]
        sched = [[1, 1], [1, 0], [0, 1], [0, 0]]
        for s in range(4):
            hu = sched[s]
            xg = [t.cpu().numpy() for t in lat]
            eng.step(lat, [s] * 2, [4] * 2, hu, g, slots)
            torch.cuda.synchronize()
            tf = pipeline.step_batch(P, cfg, [dict(x=xg[i], ctx=ctx[i], step=s, n_steps=4, has_uncond=bool(hu[i]),
                                                   g=g[i]) for i in range(2)], ctx_u, sampler)
            if sampler == "ddim":
                a, ap = sampling.ddim_alphas(4, s)
                A = np.sqrt(ap / a)
            else:
                A = 1.0
            for i in range(2):
                got = lat[i].cpu().numpy()
                r_eps = rel(got - A * xg[i], tf[i] - A * xg[i])
                kappa = 1.0
                if hu[i]:
                    t = int(sampling.timesteps(4)[s])
                    xi = xg[i] * np.float32(sampling.c_in(sampler, 4, s))
                    e = unet.forward(P, cfg, np.stack([xi, xi]), np.array([t, t]), np.stack([ctx[i], ctx_u]))
                    et = e[1] + np.float32(g[i]) * (e[0] - e[1])
                    kappa = (abs(1 - g[i]) * np.linalg.norm(e[1]) + g[i] * np.linalg.norm(e[0])) / np.linalg.norm(et)
                print(f"fp32 {sampler} step {s} req {i} cfg {hu[i]}: eps-part {r_eps:.3e} (kappa {kappa:.2f}), "
                      f"x {rel(got, tf[i]):.3e}")
                assert r_eps <= eps_part_bound(kappa, A * xg[i], tf[i] - A * xg[i]) and rel(got, tf[i]) <= TOL32
            xo = pipeline.step_batch(P, cfg, [dict(x=xo[i], ctx=ctx[i], step=s, n_steps=4, has_uncond=bool(hu[i]),
                                                   g=g[i]) for i in range(2)], ctx_u, sampler)
        final = max(rel(lat[i].cpu().numpy(), xo[i]) for i in range(2))
        print(f"fp32 {sampler} final rel-L2 {final:.3e}")
        assert final <= TOL32
    finally:
        eng.close()


def test_fp32_tiny_batch_invariance(tiny32):
    """I5 in the fp32 mode: a request's update in a ragged batch equals its update alone (bitwise)."""
    eng, P, V, ctx_u = tiny32
    ctx = [synth.text_embedding(4, i, 8, 32) for i in range(3)]
    slots = [eng.register(torch.from_numpy(c)) for c in ctx]
    x0 = [synth.initial_noise(4, i, 8, 8) for i in range(3)]
    lat = [torch.from_numpy(x).cuda() for x in x0]
    eng.step(lat, [0, 1, 2], [4, 4, 4], [1, 0, 1], [7.5, 7.5, 3.0], slots)
    for i in range(3):
        t = [torch.from_numpy(x0[i]).cuda()]
        eng.step(t, [[0, 1, 2][i]], [4], [[1, 0, 1][i]], [[7.5, 7.5, 3.0][i]], [slots[i]])
        torch.cuda.synchronize()
        assert torch.equal(lat[i], t[0]), i
    for s in slots:
        eng.release(s)


def test_fp32_tiny_vae_whole_and_chunked(tiny32):
    """CFG#1 VAE (16×16 image) in the fp32 mode: whole decode ≤ 1e-4 vs the oracle; chunked decodes
    (c = 2, 3, 5) bitwise equal to the whole decode (I6)."""
    eng, P, V, ctx_u = tiny32
    z = synth.initial_noise(2, 0, 8, 8)
    ref = vae.decode(V, configs.TINY_VAE, z[None])[0]
    zt = torch.from_numpy(z).cuda()
    whole = eng.decode(zt, 1)
    torch.cuda.synchronize()
    r = rel(whole.cpu().numpy(), ref)
    print(f"fp32 tiny VAE rel-L2 {r:.3e}")
    assert r <= TOL32
    for c in (2, 3, 5):
        ch = eng.decode(zt, c)
        torch.cuda.synchronize()
        assert torch.equal(ch, whole), c


def test_fp32_tinyxl_step():
    """SDXL code paths (added embedding, depth-2 transformers, head-dim heads) in the fp32 mode."""
    eng = Engine("tinyxl", max_latent_hw=16, b_max=4, precision="fp32")
    try:
        cfg = configs.TINY_XL_UNET
        P = configs.unet_params(cfg, 0, np.float32)
        _xl_step32(eng, cfg, P, 16, [(3, 1, 7.5), (30, 0, 7.5), (44, 1, 3.0)], 11)
    finally:
        eng.close()


def _xl_step32(eng, cfg, P, hw, spec, seed):
    n = len(spec)
    ctx_u = synth.uncond_embedding(0, cfg.ctx_len, cfg.ctx_dim)
    pu = synth.uncond_pooled(0, cfg.pooled_dim)
    eng.set_uncond(torch.from_numpy(ctx_u), torch.from_numpy(pu))
    ctx = [synth.text_embedding(seed, i, cfg.ctx_len, cfg.ctx_dim) for i in range(n)]
    pooled = [synth.pooled_embedding(seed, i, cfg.pooled_dim) for i in range(n)]
    slots = [eng.register(torch.from_numpy(c), torch.from_numpy(p)) for c, p in zip(ctx, pooled)]
    x0 = [synth.initial_noise(seed, i, hw, hw) for i in range(n)]
    lat = [torch.from_numpy(x).cuda() for x in x0]
    steps, hu, g = [r[0] for r in spec], [r[1] for r in spec], [r[2] for r in spec]
    eng.step(lat, steps, [50] * n, hu, g, slots)
    torch.cuda.synchronize()
    for i in range(n):
        t = int(sampling.timesteps(50)[steps[i]])
        eps = unet.forward(P, cfg, np.stack([x0[i], x0[i]]), np.array([t, t]), np.stack([ctx[i], ctx_u]),
                           np.stack([pooled[i], pu]))
        ec, eu = eps[0], eps[1]
        et = sampling.cfg_combine(ec, eu if hu[i] else None, g[i], bool(hu[i]))
        exp = sampling.ddim_step(x0[i], et, 50, steps[i])
        kappa = ((abs(1 - g[i]) * np.linalg.norm(eu) + g[i] * np.linalg.norm(ec)) / np.linalg.norm(et)) if hu[i] else 1.0
        a, ap = sampling.ddim_alphas(50, steps[i])
        A = np.sqrt(ap / a)
        got = lat[i].cpu().numpy()
        r_x, r_eps = rel(got, exp), rel(got - A * x0[i], exp - A * x0[i])
        print(f"fp32 {cfg.name} {hw}² req {i}: x {r_x:.3e}, eps-part {r_eps:.3e}, kappa {kappa:.2f}")
        assert r_x <= TOL32 and r_eps <= TOL32 * kappa
    for s in slots:
        eng.release(s)


def test_fp32_sd15_step_and_vae():
    """SD-1.5 shapes (all 859.5 M parameters, fp32) at latent 16×16: one ragged step (a CFG request and
    a Skip-CFG request, 3 UNet rows) and the SD VAE decode (128×128 image), each ≤ 1e-4 vs the oracle;
    chunked decode bitwise equal to the whole decode."""
    eng = Engine("sd15", max_latent_hw=16, b_max=2, precision="fp32")
    try:
        cfg = configs.SD15_UNET
        P = configs.unet_params(cfg, 0, np.float32)
        ctx_u = synth.uncond_embedding(0, 77, 768)
        eng.set_uncond(torch.from_numpy(ctx_u))
        ctx = [synth.text_embedding(2, i, 77, 768) for i in range(2)]
        slots = [eng.register(torch.from_numpy(c)) for c in ctx]
        steps, hu, g = [5, 30], [1, 0], [7.5, 7.5]
        x0 = [synth.initial_noise(2, i, 16, 16) for i in range(2)]
        lat = [torch.from_numpy(x).cuda() for x in x0]
        eng.step(lat, steps, [50, 50], hu, g, slots)
        torch.cuda.synchronize()
        ts = [int(sampling.timesteps(50)[s]) for s in steps]
        eps = unet.forward(P, cfg, np.stack([x0[0], x0[1], x0[0]]), np.array([ts[0], ts[1], ts[0]]),
                           np.stack([ctx[0], ctx[1], ctx_u]))
        for i, eu in ((0, eps[2]), (1, None)):
            ec = eps[i]
            et = sampling.cfg_combine(ec, eu, g[i], eu is not None)
            exp = sampling.ddim_step(x0[i], et, 50, steps[i])
            kappa = ((abs(1 - g[i]) * np.linalg.norm(eu) + g[i] * np.linalg.norm(ec)) / np.linalg.norm(et)) \
                if eu is not None else 1.0
            a, ap = sampling.ddim_alphas(50, steps[i])
            A = np.sqrt(ap / a)
            got = lat[i].cpu().numpy()
            r_x, r_eps = rel(got, exp), rel(got - A * x0[i], exp - A * x0[i])
            print(f"fp32 sd15 16² req {i}: x {r_x:.3e}, eps-part {r_eps:.3e}, kappa {kappa:.2f}")
            assert r_x <= TOL32 and r_eps <= TOL32 * kappa
        for s in slots:
            eng.release(s)
        V = configs.vae_params(configs.SD_VAE, 0, np.float32)
        z = synth.initial_noise(3, 0, 16, 16)
        ref = vae.decode(V, configs.SD_VAE, z[None])[0]
        zt = torch.from_numpy(z).cuda()
        whole = eng.decode(zt, 1)
        ch = eng.decode(zt, 4)
        torch.cuda.synchronize()
        r = rel(whole.cpu().numpy(), ref)
        print(f"fp32 sd VAE 128² rel-L2 {r:.3e}")
        assert r <= TOL32
        assert torch.equal(ch, whole)
    finally:
        eng.close()


def test_fp32_sdxl_step():
    """SDXL-base shapes (2.57 B parameters, fp32) at latent 32×32: one CFG request (2 UNet rows)."""
    eng = Engine("sdxl", max_latent_hw=32, b_max=1, precision="fp32")
    try:
        cfg = configs.SDXL_UNET
        P = configs.unet_params(cfg, 0, np.float32)
        _xl_step32(eng, cfg, P, 32, [(20, 1, 7.5)], 17)
    finally:
        eng.close()

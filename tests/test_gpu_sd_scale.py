"""SURVEY §8(d) SD-scale parity workload (PAPER.md:162, :230 Skip-CFG and VAE chunking; north star:
bf16 rel-L2 ≤ 2e-2 on final latents AND images): SD-1.5 at 512² (latent 64×64), two requests in one
continuous batch — n = 4 with one Skip-CFG step and n = 6 with CFG on every step, both g = 7.5 — the
first finishing early and leaving the second to run on alone; each finished latent is decoded in two
chunks on a low-priority stream while the other request's UNet steps run on the high-priority one.
Everything goes through the C ABI; the oracle runs each request alone (I5) with the same skip set and
decodes its final latent whole (I6 makes the chunked GPU decode comparable to it).

A second test compares the UNet ε of EVERY row of a ragged SD-1.5 step — ε_c and ε_u separately,
each at 2e-2 (sd_debug_step_eps) — so the CFG amplification κ of the combine never loosens a bound."""
import numpy as np
import pytest
import torch

import synth
from oracle import configs, pipeline, sampling, unet, vae

pytestmark = pytest.mark.gpu

from paper_2605_08835_b200.engine import Engine  # noqa: E402

TOL = 2e-2


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module", params=["bf16", "fp16"])
def sd15(request):
    eng = Engine("sd15", max_latent_hw=64, b_max=4, c_max=4, precision=request.param)
    ctx_u = synth.uncond_embedding(0, 77, 768)
    eng.set_uncond(torch.from_numpy(ctx_u))
    P = configs.unet_params(configs.SD15_UNET, 0, np.float32, bf16_weights=True)
    yield eng, P, synth.bf16_round(ctx_u)
    eng.close()


@pytest.mark.timeout(1800)
def test_sd15_512_two_requests_skip_cfg_two_chunk_vae(sd15):
    eng, P, ctx_u = sd15
    n_steps = [4, 6]
    skips = [{2}, set()]
    g = [7.5, 7.5]
    seed = 41
    ctx = [synth.text_embedding(seed, i, 77, 768) for i in range(2)]
    slots = [eng.register(torch.from_numpy(c)) for c in ctx]
    xT = [synth.initial_noise(seed, i, 64, 64) for i in range(2)]
    lat = [torch.from_numpy(x * np.float32(eng.init_sigma(n))).cuda() for x, n in zip(xT, n_steps)]
    hi = torch.cuda.Stream(priority=-1)
    lo = torch.cuda.Stream(priority=0)
    imgs = [torch.empty(3, 512, 512, device="cuda") for _ in range(2)]
    dec_state = [None, None]
    import ctypes as C
    for s in range(max(n_steps)):
        act = [i for i in range(2) if s < n_steps[i]]
        with torch.cuda.stream(hi):
            eng.step([lat[i] for i in act], [s] * len(act), [n_steps[i] for i in act],
                     [0 if s in skips[i] else 1 for i in act], [g[i] for i in act], [slots[i] for i in act],
                     stream=hi)
        # request 0 exits after step 3: its 2-chunk decode runs one chunk per round on the low-priority
        # stream, concurrently with request 1's remaining UNet rounds (R9 / Eq. 2)
        if s + 1 == n_steps[0]:
            lo.wait_stream(hi)
            dec_state[0] = C.c_void_p()
        elif s >= n_steps[0] and dec_state[0] is not None:
            j = s - n_steps[0]
            if j < 2:
                eng.decode_chunk(lat[0], 2, j, dec_state[0], imgs[0], stream=lo)
    lo.wait_stream(hi)
    st1 = C.c_void_p()
    for j in range(2):
        eng.decode_chunk(lat[1], 2, j, st1, imgs[1], stream=lo)
    torch.cuda.synchronize()
    for sl in slots:
        eng.release(sl)
    V = configs.vae_params(configs.SD_VAE, 0, np.float32, bf16_weights=True)
    worst = 0.0
    for i in range(2):
        x = pipeline.denoise(P, configs.SD15_UNET, xT[i], synth.bf16_round(ctx[i]), ctx_u, n_steps[i], g[i], "ddim",
                             skip=skips[i])
        img = vae.decode(V, configs.SD_VAE, x[None])[0]
        r_x = rel(lat[i].cpu().numpy(), x)
        r_img = rel(imgs[i].cpu().numpy(), img)
        print(f"sd15 512² {eng.precision} request {i} (n {n_steps[i]}, skip {sorted(skips[i])}): final latent rel-L2 {r_x:.3e}, "
              f"image rel-L2 {r_img:.3e} (bound {TOL})")
        worst = max(worst, r_x, r_img)
    assert worst <= TOL


def test_sd15_per_row_eps(sd15):
    """ε_c and ε_u of every row of a ragged step (two CFG requests + one Skip-CFG: 5 rows), each vs the
    oracle's ε of the same row at 2e-2 — no κ factor."""
    eng, P, ctx_u = sd15
    cfg = configs.SD15_UNET
    ctx = [synth.text_embedding(43, i, 77, 768) for i in range(3)]
    slots = [eng.register(torch.from_numpy(c)) for c in ctx]
    steps, hu, g = [0, 20, 45], [1, 0, 1], [7.5, 7.5, 4.0]
    x0 = [synth.initial_noise(43, i, 64, 64) for i in range(3)]
    lat = [torch.from_numpy(x).cuda() for x in x0]
    eps = eng.step_eps(lat, steps, [50] * 3, hu, g, slots)
    torch.cuda.synchronize()
    got = eps.cpu().numpy()
    assert all(np.array_equal(lat[i].cpu().numpy(), x0[i]) for i in range(3))   # latents untouched
    cb = [synth.bf16_round(c) for c in ctx]
    ts = [int(sampling.timesteps(50)[s]) for s in steps]
    order = [0, 1, 2, 0, 2]       # R26: cond rows, then uncond rows of the CFG requests
    ref = unet.forward(P, cfg, np.stack([x0[i] for i in order]), np.array([ts[i] for i in order]),
                       np.stack([cb[0], cb[1], cb[2], ctx_u, ctx_u]))
    errs = [rel(got[k], ref[k]) for k in range(5)]
    print(f"sd15 {eng.precision} per-row eps rel-L2 (c0, c1, c2, u0, u2): " + ", ".join(f"{e:.3e}" for e in errs))
    for s in slots:
        eng.release(s)
    assert max(errs) <= TOL

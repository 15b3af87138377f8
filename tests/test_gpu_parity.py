"""End-to-end parity of the CUDA path (through the C ABI) against the NumPy oracle on the same seeded
inputs (north star tolerances: bf16 rel-L2 ≤ 2e-2 on latents and images).

The oracle uses the bf16-rounded weights the GPU stores (R20) and the bf16-rounded text embedding
(the GPU computes the text K/V from a bf16 copy); everything else in the oracle is fp32."""
import ctypes as C

import numpy as np
import pytest
import torch

import synth
from oracle import configs, pipeline, sampling, unet, vae

pytestmark = pytest.mark.gpu

from paper_2605_08835_b200.engine import Engine  # noqa: E402

TOL = 2e-2


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module", params=["bf16", "fp16"])
def tiny(request):
    eng = Engine("tiny", max_latent_hw=16, b_max=4, precision=request.param)
    ctx_u = synth.uncond_embedding(0, 8, 32)
    eng.set_uncond(torch.from_numpy(ctx_u))
    P = configs.unet_params(configs.TINY_UNET, 0, np.float32, bf16_weights=True)
    V = configs.vae_params(configs.TINY_VAE, 0, np.float32, bf16_weights=True)
    yield eng, P, V, synth.bf16_round(ctx_u)
    eng.close()


def _cfg_gain(P, x, t, ctx, ctx_u, g):
    """Error-propagation factor of the CFG combine for one request: ε̃ = (1−g)ε_u + g ε_c, so a
    relative kernel error δ on ε_c and ε_u becomes ≤ κ·δ on ε̃ with
    κ = (|1−g|·‖ε_u‖ + g·‖ε_c‖) / ‖ε̃‖ (tolerance derivation)."""
    e = unet.forward(P, configs.TINY_UNET, np.stack([x, x]), np.array([t, t]), np.stack([ctx, ctx_u]))
    ec, eu = e[0], e[1]
    et = eu + np.float32(g) * (ec - eu)
    return (abs(1 - g) * np.linalg.norm(eu) + g * np.linalg.norm(ec)) / np.linalg.norm(et)


def _run_tiny(eng, P, ctx_u, sampler, schedule, g=(7.5, 5.0)):
    """schedule[s] = per-request has_uncond at step s; both requests 4 steps. Returns the final
    rel-L2 vs the free-running oracle and, per step, the teacher-forced ε-part error divided by
    its allowed bound (TOL for cond-only steps, TOL·κ for CFG steps)."""
    n = len(g)
    ctx = [synth.text_embedding(1, i, 8, 32) for i in range(n)]
    slots = [eng.register(torch.from_numpy(c)) for c in ctx]
    sig = sampling.init_sigma(sampler, 4)
    assert abs(eng.init_sigma(4) - sig) < 1e-6
    x0 = [synth.initial_noise(1, i, 8, 8) * np.float32(sig) for i in range(n)]
    lat = [torch.from_numpy(x).cuda() for x in x0]
    xo = [x.copy() for x in x0]
    worst = 0.0
    for s in range(4):
        hu = schedule[s]
        xg = [t.cpu().numpy() for t in lat]
        eng.step(lat, [s] * n, [4] * n, hu, list(g), slots)
        torch.cuda.synchronize()
        cb = [synth.bf16_round(c) for c in ctx]
        reqs_tf = [dict(x=xg[i], ctx=cb[i], step=s, n_steps=4, has_uncond=bool(hu[i]), g=g[i]) for i in range(n)]
        tf = pipeline.step_batch(P, configs.TINY_UNET, reqs_tf, ctx_u, sampler)
        a, ap = sampling.ddim_alphas(4, s)
        A = np.sqrt(ap / a) if sampler == "ddim" else 1.0
        t = int(sampling.timesteps(4)[s])
        for i in range(n):
            got = lat[i].cpu().numpy()
            r_eps = rel(got - A * xg[i], tf[i] - A * xg[i])        # ε-part of the update (R21)
            kappa = _cfg_gain(P, xg[i] * np.float32(sampling.c_in(sampler, 4, s)), t, cb[i], ctx_u, g[i]) \
                if hu[i] else 1.0
            print(f"  step {s} req {i} cfg={hu[i]} eps-part rel {r_eps:.3e} (kappa {kappa:.2f}) x rel "
                  f"{rel(got, tf[i]):.3e}")
            worst = max(worst, r_eps / (TOL * kappa), rel(got, tf[i]) / TOL)
        reqs = [dict(x=xo[i], ctx=cb[i], step=s, n_steps=4, has_uncond=bool(hu[i]), g=g[i]) for i in range(n)]
        xo = pipeline.step_batch(P, configs.TINY_UNET, reqs, ctx_u, sampler)
    final = max(rel(lat[i].cpu().numpy(), xo[i]) for i in range(n))
    for sl in slots:
        eng.release(sl)
    return final, worst, lat, xo


@pytest.mark.parametrize("sampler", ["ddim"])
def test_tiny_unet_cfg_on_off(tiny, sampler):
    eng, P, V, ctx_u = tiny
    sched = [[1, 1], [1, 0], [0, 1], [0, 0]]     # CFG on / Skip-CFG mixes (CFG#1)
    final, worst, lat, xo = _run_tiny(eng, P, ctx_u, sampler, sched)
    print(f"tiny {eng.precision} final rel-L2 {final:.3e}, worst per-step error / bound {worst:.3f}")
    assert final <= TOL and worst <= 1.0


@pytest.mark.parametrize("precision", ["bf16", "fp16"])
def test_tiny_unet_ln_fold(precision, monkeypatch):
    """The folded-LayerNorm engine path (SD_LN_FOLD=1: LN1/LN2/LN3 applied in the q|k|v, Vt, q2 and FF1 GEMM
    epilogues) against the oracle on the CFG / Skip-CFG schedule of test_tiny_unet_cfg_on_off."""
    monkeypatch.setenv("SD_LN_FOLD", "1")
    eng = Engine("tiny", max_latent_hw=16, b_max=4, precision=precision)
    try:
        ctx_u = synth.uncond_embedding(0, 8, 32)
        eng.set_uncond(torch.from_numpy(ctx_u))
        P = configs.unet_params(configs.TINY_UNET, 0, np.float32, bf16_weights=True)
        final, worst, _, _ = _run_tiny(eng, P, synth.bf16_round(ctx_u), "ddim", [[1, 1], [1, 0], [0, 1], [0, 0]])
        print(f"tiny {precision} LN-fold final rel-L2 {final:.3e}, worst per-step error / bound {worst:.3f}")
        assert final <= TOL and worst <= 1.0
    finally:
        eng.close()


def test_tiny_unet_euler():
    """R5 Euler (ε-prediction, σ grid on the same timesteps) through the bf16 path: 4 steps with CFG /
    Skip-CFG mixes vs the oracle (final latents and teacher-forced ε-parts)."""
    eng = Engine("tiny", max_latent_hw=16, b_max=4, sampler="euler")
    try:
        ctx_u = synth.uncond_embedding(0, 8, 32)
        eng.set_uncond(torch.from_numpy(ctx_u))
        P = configs.unet_params(configs.TINY_UNET, 0, np.float32, bf16_weights=True)
        final, worst, _, _ = _run_tiny(eng, P, synth.bf16_round(ctx_u), "euler", [[1, 1], [1, 0], [0, 1], [0, 0]])
        print(f"tiny Euler final rel-L2 {final:.3e}, worst per-step error / bound {worst:.3f}")
        assert final <= TOL and worst <= 1.0
    finally:
        eng.close()


def test_tiny_batch_invariance(tiny):
    """I5 on the GPU: a request's update in a batch equals its update alone (bitwise)."""
    eng, P, V, ctx_u = tiny
    ctx = [synth.text_embedding(4, i, 8, 32) for i in range(3)]
    slots = [eng.register(torch.from_numpy(c)) for c in ctx]
    x0 = [synth.initial_noise(4, i, 8, 8) for i in range(3)]
    lat = [torch.from_numpy(x).cuda() for x in x0]
    eng.step(lat, [0, 1, 2], [4, 4, 4], [1, 0, 1], [7.5, 7.5, 3.0], slots)
    alone = []
    for i in range(3):
        t = [torch.from_numpy(x0[i]).cuda()]
        eng.step(t, [[0, 1, 2][i]], [4], [[1, 0, 1][i]], [[7.5, 7.5, 3.0][i]], [slots[i]])
        alone.append(t[0])
    torch.cuda.synchronize()
    for i in range(3):
        assert torch.equal(lat[i], alone[i]), i
    for s in slots:
        eng.release(s)


def test_tiny_vae_whole_and_chunked(tiny):
    eng, P, V, ctx_u = tiny
    z = synth.initial_noise(2, 0, 8, 8)
    ref = vae.decode(V, configs.TINY_VAE, z[None].astype(np.float32))[0]
    zt = torch.from_numpy(z).cuda()
    whole = eng.decode(zt, 1)
    torch.cuda.synchronize()
    r = rel(whole.cpu().numpy(), ref)
    print(f"tiny {eng.precision} VAE rel-L2 {r:.3e}")
    assert r <= TOL
    for c in (2, 3, 5):
        ch = eng.decode(zt, c)
        torch.cuda.synchronize()
        assert torch.equal(ch, whole), c                 # I6 on the GPU: bitwise


def test_vae_chunk_order_enforced(tiny):
    eng, *_ = tiny
    from paper_2605_08835_b200 import binding as B
    z = torch.zeros(4, 8, 8, device="cuda")
    img = torch.empty(3, 64, 64, device="cuda")
    st = C.c_void_p()
    with pytest.raises(B.SDError) as ei:
        eng.decode_chunk(z, 3, 1, st, img)
    assert ei.value.status in (B.SD_E_STATE, B.SD_E_INVAL)


@pytest.fixture(scope="module", params=["bf16", "fp16"])
def sd15(request):
    eng = Engine("sd15", max_latent_hw=64, b_max=8, precision=request.param)
    ctx_u = synth.uncond_embedding(0, 77, 768)
    eng.set_uncond(torch.from_numpy(ctx_u))
    yield eng, synth.bf16_round(ctx_u)
    eng.close()


def test_sd15_step_parity(sd15):
    """One ragged SD-1.5 512² step (3 requests, 5 rows: two CFG requests + one Skip-CFG) vs the oracle.
    Bounds: final-step x at TOL; ε-part at TOL·κ_r (κ = CFG error-propagation factor)."""
    eng, ctx_u = sd15
    cfg = configs.SD15_UNET
    P = configs.unet_params(cfg, 0, np.float32, bf16_weights=True)
    ctx = [synth.text_embedding(1, i, 77, 768) for i in range(3)]
    slots = [eng.register(torch.from_numpy(c)) for c in ctx]
    steps, hu, g = [0, 20, 45], [1, 0, 1], [7.5, 7.5, 4.0]
    x0 = [synth.initial_noise(1, i, 64, 64) for i in range(3)]
    lat = [torch.from_numpy(x).cuda() for x in x0]
    eng.step(lat, steps, [50] * 3, hu, g, slots)
    torch.cuda.synchronize()
    # oracle: the five rows of this step (R26: cond rows, then uncond rows)
    cb = [synth.bf16_round(c) for c in ctx]
    ts = [int(sampling.timesteps(50)[s]) for s in steps]
    rows_x = np.stack([x0[0], x0[1], x0[2], x0[0], x0[2]])
    rows_t = np.array([ts[0], ts[1], ts[2], ts[0], ts[2]])
    rows_c = np.stack([cb[0], cb[1], cb[2], ctx_u, ctx_u])
    eps = unet.forward(P, cfg, rows_x, rows_t, rows_c)
    unc = {0: 3, 2: 4}
    worst = 0.0
    for i in range(3):
        ec = eps[i]
        eu = eps[unc[i]] if hu[i] else None
        et = sampling.cfg_combine(ec, eu, g[i], bool(hu[i]))
        exp = sampling.ddim_step(x0[i], et, 50, steps[i])
        kappa = ((abs(1 - g[i]) * np.linalg.norm(eu) + g[i] * np.linalg.norm(ec)) / np.linalg.norm(et)) if hu[i] else 1.0
        a, ap = sampling.ddim_alphas(50, steps[i])
        A = np.sqrt(ap / a)
        got = lat[i].cpu().numpy()
        r_x = rel(got, exp)
        r_eps = rel(got - A * x0[i], exp - A * x0[i])      # ε-part (R21)
        print(f"sd15 {eng.precision} req {i} (step {steps[i]}, cfg {hu[i]}, g {g[i]}): x rel-L2 {r_x:.3e}, eps-part rel-L2 "
              f"{r_eps:.3e}, kappa {kappa:.2f}, eps-part/kappa {r_eps / kappa:.3e}")
        worst = max(worst, r_x / TOL, r_eps / (TOL * kappa))
    for s in slots:
        eng.release(s)
    assert worst <= 1.0


def test_sd15_vae_parity(sd15):
    eng, _ = sd15
    V = configs.vae_params(configs.SD_VAE, 0, np.float32, bf16_weights=True)
    z = synth.initial_noise(3, 0, 64, 64)
    ref = vae.decode(V, configs.SD_VAE, z[None])[0]
    zt = torch.from_numpy(z).cuda()
    whole = eng.decode(zt, 1)
    ch = eng.decode(zt, 4)
    torch.cuda.synchronize()
    r = rel(whole.cpu().numpy(), ref)
    print(f"sd VAE {eng.precision} 512² rel-L2 {r:.3e}")
    assert r <= TOL
    assert torch.equal(ch, whole)


def test_sd15_768_step_and_vae_parity():
    """CFG#4 resolution: SD-1.5 at 768² (latent 96×96: self-attention over 9216 / 2304 tokens on the
    tcgen05 path, 576 / 144 on the mma path; conv tiles of 32×4 px). One CFG request, one step, vs
    the oracle (ε-part at TOL·κ, x at TOL), then the 768² VAE decode (TOL) and chunked == whole."""
    eng = Engine("sd15", max_latent_hw=96, b_max=1)
    try:
        ctx_u = synth.uncond_embedding(0, 77, 768)
        eng.set_uncond(torch.from_numpy(ctx_u))
        cfg = configs.SD15_UNET
        P = configs.unet_params(cfg, 0, np.float32, bf16_weights=True)
        ctx = synth.text_embedding(5, 0, 77, 768)
        slot = eng.register(torch.from_numpy(ctx))
        x0 = synth.initial_noise(5, 0, 96, 96)
        lat = [torch.from_numpy(x0).cuda()]
        step, g = 10, 7.5
        eng.step(lat, [step], [50], [1], [g], [slot])
        torch.cuda.synchronize()
        t = int(sampling.timesteps(50)[step])
        eps = unet.forward(P, cfg, np.stack([x0, x0]), np.array([t, t]),
                           np.stack([synth.bf16_round(ctx), synth.bf16_round(ctx_u)]))
        ec, eu = eps[0], eps[1]
        et = sampling.cfg_combine(ec, eu, g, True)
        exp = sampling.ddim_step(x0, et, 50, step)
        kappa = (abs(1 - g) * np.linalg.norm(eu) + g * np.linalg.norm(ec)) / np.linalg.norm(et)
        a, ap = sampling.ddim_alphas(50, step)
        A = np.sqrt(ap / a)
        got = lat[0].cpu().numpy()
        r_x, r_eps = rel(got, exp), rel(got - A * x0, exp - A * x0)
        print(f"sd15 768²: x rel-L2 {r_x:.3e}, eps-part {r_eps:.3e}, kappa {kappa:.2f}")
        assert r_x <= TOL and r_eps <= TOL * kappa
        V = configs.vae_params(configs.SD_VAE, 0, np.float32, bf16_weights=True)
        z = synth.initial_noise(6, 0, 96, 96)
        ref = vae.decode(V, configs.SD_VAE, z[None])[0]
        zt = torch.from_numpy(z).cuda()
        whole = eng.decode(zt, 1)
        ch = eng.decode(zt, 3)
        torch.cuda.synchronize()
        r = rel(whole.cpu().numpy(), ref)
        print(f"sd VAE 768² rel-L2 {r:.3e}")
        assert r <= TOL
        assert torch.equal(ch, whole)
        eng.release(slot)
    finally:
        eng.close()


def _xl_step_check(eng, cfg, P, lat_hw, reqs_spec, seed):
    """One ragged step of an SDXL-shaped engine vs the oracle: reqs_spec = [(step, has_uncond, g)];
    ε-part at TOL·κ, x at TOL."""
    n = len(reqs_spec)
    ctx_u = synth.uncond_embedding(0, cfg.ctx_len, cfg.ctx_dim)
    pu = synth.uncond_pooled(0, cfg.pooled_dim)
    eng.set_uncond(torch.from_numpy(ctx_u), torch.from_numpy(pu))
    ctx = [synth.text_embedding(seed, i, cfg.ctx_len, cfg.ctx_dim) for i in range(n)]
    pooled = [synth.pooled_embedding(seed, i, cfg.pooled_dim) for i in range(n)]
    slots = [eng.register(torch.from_numpy(c), torch.from_numpy(p)) for c, p in zip(ctx, pooled)]
    x0 = [synth.initial_noise(seed, i, lat_hw, lat_hw) for i in range(n)]
    lat = [torch.from_numpy(x).cuda() for x in x0]
    steps = [r[0] for r in reqs_spec]
    hu = [r[1] for r in reqs_spec]
    g = [r[2] for r in reqs_spec]
    eng.step(lat, steps, [50] * n, hu, g, slots)
    torch.cuda.synchronize()
    cb = [synth.bf16_round(c) for c in ctx]
    cub = synth.bf16_round(ctx_u)
    worst = 0.0
    for i in range(n):
        t = int(sampling.timesteps(50)[steps[i]])
        rx = np.stack([x0[i], x0[i]])
        eps = unet.forward(P, cfg, rx, np.array([t, t]), np.stack([cb[i], cub]), np.stack([pooled[i], pu]))
        ec, eu = eps[0], eps[1]
        et = sampling.cfg_combine(ec, eu if hu[i] else None, g[i], bool(hu[i]))
        exp = sampling.ddim_step(x0[i], et, 50, steps[i])
        kappa = ((abs(1 - g[i]) * np.linalg.norm(eu) + g[i] * np.linalg.norm(ec)) / np.linalg.norm(et)) if hu[i] else 1.0
        a, ap = sampling.ddim_alphas(50, steps[i])
        A = np.sqrt(ap / a)
        got = lat[i].cpu().numpy()
        r_x, r_eps = rel(got, exp), rel(got - A * x0[i], exp - A * x0[i])
        print(f"{cfg.name} {lat_hw}² req {i} (step {steps[i]}, cfg {hu[i]}): x {r_x:.3e}, eps-part {r_eps:.3e}, "
              f"kappa {kappa:.2f}")
        worst = max(worst, r_x / TOL, r_eps / (TOL * kappa))
    for s in slots:
        eng.release(s)
    return worst


def test_tinyxl_step_parity():
    """SDXL code paths at tiny size: no attention at level 0, depth-2 transformers, head-dim heads,
    linear projections, the added (pooled ‖ time ids) embedding per prompt slot."""
    eng = Engine("tinyxl", max_latent_hw=16, b_max=4)
    try:
        P = configs.unet_params(configs.TINY_XL_UNET, 0, np.float32, bf16_weights=True)
        worst = _xl_step_check(eng, configs.TINY_XL_UNET, P, 16, [(3, 1, 7.5), (30, 0, 7.5), (44, 1, 3.0)], 11)
        assert worst <= 1.0
    finally:
        eng.close()


def test_sdxl_step_and_vae_parity():
    """SDXL-base shapes (2.57 B parameters) at latent 64×64: self-attention on the tcgen05 path at
    d = 64 (1024 / 256 tokens), cross-attention to 77×2048 text, the 10-block transformers; then the
    SDXL VAE (scaling factor 0.13025) at latent 32×32."""
    eng = Engine("sdxl", max_latent_hw=64, b_max=2)
    try:
        P = configs.unet_params(configs.SDXL_UNET, 0, np.float32, bf16_weights=True)
        worst = _xl_step_check(eng, configs.SDXL_UNET, P, 64, [(12, 1, 7.5), (40, 0, 5.0)], 13)
        assert worst <= 1.0
        V = configs.vae_params(configs.SDXL_VAE, 0, np.float32, bf16_weights=True)
        z = synth.initial_noise(8, 0, 32, 32)
        ref = vae.decode(V, configs.SDXL_VAE, z[None])[0]
        img = eng.decode(torch.from_numpy(z).cuda(), 1)
        torch.cuda.synchronize()
        r = rel(img.cpu().numpy(), ref)
        print(f"sdxl VAE 256² rel-L2 {r:.3e}")
        assert r <= TOL
    finally:
        eng.close()


def test_sd15_bench_launch_config(sd15):
    """The launch configuration bench.py times (CFG#2: 8 requests in lockstep, CFG on every row → 16
    UNet rows at latent 64×64). The oracle cannot run all 16 rows in seconds, so: request 0 is checked
    against the oracle (its cond + uncond rows; ε-part at TOL·κ, x at TOL), and every other request's
    update inside the 16-row batch must equal its update alone bitwise (I5), which pins each of them to
    the oracle-checked single-request path."""
    eng, ctx_u = sd15
    cfg = configs.SD15_UNET
    n, step, g = 8, 7, 7.5
    ctx = [synth.text_embedding(9, i, 77, 768) for i in range(n)]
    slots = [eng.register(torch.from_numpy(c)) for c in ctx]
    x0 = [synth.initial_noise(9, i, 64, 64) for i in range(n)]
    lat = [torch.from_numpy(x).cuda() for x in x0]
    eng.step(lat, [step] * n, [50] * n, [1] * n, [g] * n, slots)
    torch.cuda.synchronize()
    for i in (3, 7):
        alone = [torch.from_numpy(x0[i]).cuda()]
        eng.step(alone, [step], [50], [1], [g], [slots[i]])
        torch.cuda.synchronize()
        assert torch.equal(alone[0], lat[i]), i
    P = configs.unet_params(cfg, 0, np.float32, bf16_weights=True)
    t = int(sampling.timesteps(50)[step])
    eps = unet.forward(P, cfg, np.stack([x0[0], x0[0]]), np.array([t, t]),
                       np.stack([synth.bf16_round(ctx[0]), ctx_u]))
    ec, eu = eps[0], eps[1]
    et = sampling.cfg_combine(ec, eu, g, True)
    exp = sampling.ddim_step(x0[0], et, 50, step)
    kappa = (abs(1 - g) * np.linalg.norm(eu) + g * np.linalg.norm(ec)) / np.linalg.norm(et)
    a, ap = sampling.ddim_alphas(50, step)
    A = np.sqrt(ap / a)
    got = lat[0].cpu().numpy()
    r_x, r_eps = rel(got, exp), rel(got - A * x0[0], exp - A * x0[0])
    print(f"sd15 {eng.precision} 16-row bench launch, request 0: x {r_x:.3e}, eps-part {r_eps:.3e}, kappa {kappa:.2f}")
    for s in slots:
        eng.release(s)
    assert r_x <= TOL and r_eps <= TOL * kappa


def test_sdxl_1024_full_size_properties():
    """CFG#5 at its full size (SDXL-base, 1024², latent 128×128), where the oracle cannot run in seconds:
    properties that hold at any size. (1) A ragged 2-request step (one CFG, one Skip-CFG; 3 UNet rows)
    equals each request stepped alone, bitwise (I5). (2) The 1024² decode chunked into c = 4, 8, 16
    work-item ranges equals the whole decode bitwise (I6, the paper's 4-16 chunk sweep). (3) Outputs
    are finite and the decoded image is not constant."""
    eng = Engine("sdxl", max_latent_hw=128, b_max=2, c_max=16)
    try:
        cfg = configs.SDXL_UNET
        ctx_u = synth.uncond_embedding(0, cfg.ctx_len, cfg.ctx_dim)
        pu = synth.uncond_pooled(0, cfg.pooled_dim)
        eng.set_uncond(torch.from_numpy(ctx_u), torch.from_numpy(pu))
        ctx = [synth.text_embedding(21, i, cfg.ctx_len, cfg.ctx_dim) for i in range(2)]
        pooled = [synth.pooled_embedding(21, i, cfg.pooled_dim) for i in range(2)]
        slots = [eng.register(torch.from_numpy(c), torch.from_numpy(p)) for c, p in zip(ctx, pooled)]
        x0 = [synth.initial_noise(21, i, 128, 128) for i in range(2)]
        lat = [torch.from_numpy(x).cuda() for x in x0]
        steps, hu, g = [10, 40], [1, 0], [7.5, 7.5]
        eng.step(lat, steps, [50, 50], hu, g, slots)
        for i in range(2):
            alone = [torch.from_numpy(x0[i]).cuda()]
            eng.step(alone, [steps[i]], [50], [hu[i]], [g[i]], [slots[i]])
            torch.cuda.synchronize()
            assert torch.equal(alone[0], lat[i]), i
            assert torch.isfinite(lat[i]).all()
        whole = eng.decode(lat[0], 1)
        torch.cuda.synchronize()
        assert whole.shape == (3, 1024, 1024) and torch.isfinite(whole).all() and whole.std() > 1e-3
        for c in (4, 8, 16):
            ch = eng.decode(lat[0], c)
            torch.cuda.synchronize()
            assert torch.equal(ch, whole), c
        for s in slots:
            eng.release(s)
    finally:
        eng.close()


def test_vae_tiled_v2(tiny):
    """V2 independent tiles (R7 V2) on the GPU: equals the oracle's decode_tiled
    on the same inputs (north-star 2e-2); reproduces the whole decode bitwise when the tile or the
    halo covers the latent; and with a small halo it is the approximation it is meant to be (error
    vs the whole decode > 0, shrinking as the halo grows)."""
    eng, P, V, ctx_u = tiny
    z = synth.initial_noise(7, 0, 16, 16)
    zt = torch.from_numpy(z).cuda()
    whole = eng.decode(zt, 1)
    torch.cuda.synchronize()
    assert torch.equal(eng.decode_tiled(zt, 16, 0), whole)
    assert torch.equal(eng.decode_tiled(zt, 8, 8), whole)       # every window is the whole latent
    errs = []
    for halo in (0, 8):
        t = eng.decode_tiled(zt, 8, halo)
        torch.cuda.synchronize()
        errs.append(rel(t.cpu().numpy(), whole.cpu().numpy()))
    ref = vae.decode_tiled(V, configs.TINY_VAE, z[None], tile=8, halo=0)[0]
    got = eng.decode_tiled(zt, 8, 0)
    torch.cuda.synchronize()
    r = rel(got.cpu().numpy(), ref)
    print(f"tiled V2 tiny: vs oracle {r:.3e}; error vs whole decode halo 0: {errs[0]:.3e}, halo 8: {errs[1]:.3e}")
    assert r <= TOL
    assert errs[0] > 1e-3 and errs[1] == 0.0


def test_vae_tiled_v2_sd_shape(sd15):
    """V2 on the SD VAE at latent 32×32 (256² image): vs the oracle's decode_tiled (tile 16, halo 8;
    four 24×24 windows) within 2e-2, and bitwise equal to the whole decode when tile ≥ latent."""
    eng, _ = sd15
    V = configs.vae_params(configs.SD_VAE, 0, np.float32, bf16_weights=True)
    z = synth.initial_noise(7, 1, 32, 32)
    zt = torch.from_numpy(z).cuda()
    whole = eng.decode(zt, 1)
    torch.cuda.synchronize()
    assert torch.equal(eng.decode_tiled(zt, 32, 8), whole)
    got = eng.decode_tiled(zt, 16, 8)
    torch.cuda.synchronize()
    ref = vae.decode_tiled(V, configs.SD_VAE, z[None], tile=16, halo=8)[0]
    r = rel(got.cpu().numpy(), ref)
    e = rel(got.cpu().numpy(), whole.cpu().numpy())
    print(f"tiled V2 SD 32²: vs oracle {r:.3e}; vs whole decode {e:.3e}")
    assert r <= TOL


@pytest.mark.parametrize("model", ["tiny", "tinyxl"])
def test_set_weight_every_parameter(model):
    """sd_engine_set_weight: EVERY oracle parameter of a seed-7 model is loaded into a
    seed-0 engine by name in its PyTorch layout; one ragged step's per-row ε and a 2-chunk decode then
    match the seed-7 oracle — so every name, layout transform (conv tap-major, GEGLU interleave, the
    fused temb / text-K/V rows, padded channels) round-trips. Unknown names and wrong sizes are rejected."""
    from paper_2605_08835_b200 import binding as B
    ucfg = configs.TINY_UNET if model == "tiny" else configs.TINY_XL_UNET
    vcfg = configs.TINY_VAE
    eng = Engine(model, max_latent_hw=8, b_max=4, weight_seed=0)
    try:
        P7 = configs.unet_params(ucfg, 7, np.float32, bf16_weights=True)
        V7 = configs.vae_params(vcfg, 7, np.float32, bf16_weights=True)
        for name, val in list(P7.items()) + list(V7.items()):
            eng.set_weight(name, val)
        with pytest.raises(B.SDError):
            eng.set_weight("no.such.parameter", np.zeros(4, np.float32))
        with pytest.raises(B.SDError):
            eng.set_weight("conv_in.bias", np.zeros(3, np.float32))
        xl = ucfg.pooled_dim > 0
        ctx_u = synth.uncond_embedding(0, ucfg.ctx_len, ucfg.ctx_dim)
        pu = synth.uncond_pooled(0, ucfg.pooled_dim) if xl else None
        eng.set_uncond(torch.from_numpy(ctx_u), torch.from_numpy(pu) if xl else None)
        ctx = [synth.text_embedding(9, i, ucfg.ctx_len, ucfg.ctx_dim) for i in range(2)]
        pc = [synth.pooled_embedding(9, i, ucfg.pooled_dim) if xl else None for i in range(2)]
        slots = [eng.register(torch.from_numpy(c), torch.from_numpy(p) if xl else None) for c, p in zip(ctx, pc)]
        x0 = [synth.initial_noise(9, i, 8, 8) for i in range(2)]
        lat = [torch.from_numpy(x).cuda() for x in x0]
        eps = eng.step_eps(lat, [0, 2], [4, 4], [1, 0], [7.5, 7.5], slots)
        z = synth.initial_noise(9, 5, 8, 8)
        img = eng.decode(torch.from_numpy(z).cuda(), 2)
        torch.cuda.synchronize()
        ts = sampling.timesteps(4)
        order = [0, 1, 0]                       # R26: cond rows (requests 0, 1), then request 0's uncond row
        cb = [synth.bf16_round(ctx[0]), synth.bf16_round(ctx[1]), synth.bf16_round(ctx_u)]
        pooled = np.stack([pc[0], pc[1], pu]) if xl else None
        ref = unet.forward(P7, ucfg, np.stack([x0[i] for i in order]), np.array([ts[0], ts[2], ts[0]]),
                           np.stack(cb), pooled)
        got = eps.cpu().numpy()
        errs = [rel(got[k], ref[k]) for k in range(3)]
        r_img = rel(img.cpu().numpy(), vae.decode(V7, vcfg, z[None])[0])
        print(f"{model} set_weight: per-row eps rel-L2 {['%.2e' % e for e in errs]}, image {r_img:.2e}")
        assert max(errs) <= TOL and r_img <= TOL
        for s in slots:
            eng.release(s)
    finally:
        eng.close()

"""Pins for oracle/unet.py, oracle/vae.py, oracle/sampling.py and the whole-request pipeline.

No paper value pins the UNet (random weights, PAPER.md names only "SDv1.5"); it is pinned
structurally plus by the public SD-1.5 parameter count."""
import numpy as np
import pytest

import synth
from oracle import configs, pipeline, sampling, unet, vae

T = configs.TINY_UNET
TV = configs.TINY_VAE


@pytest.fixture(scope="module")
def P64():
    return configs.unet_params(T, 0, np.float64)


@pytest.fixture(scope="module")
def V64():
    return configs.vae_params(TV, 0, np.float64)


def test_sd15_param_count():
    # diffusers SD-1.5 UNet2DConditionModel has 859,520,964 parameters (public model card count)
    n = sum(int(np.prod(s[1])) for s in configs.unet_param_specs(configs.SD15_UNET))
    assert n == 859_520_964


def test_sd_vae_param_count():
    """The SD AutoencoderKL has 83,653,863 parameters (the widely published count). The oracle builds
    only post_quant_conv + decoder; the encoder + quant_conv side is counted here from the standard
    SD encoder layout (conv_in 3→128; down blocks 128/256/512/512 × 2 ResNets, 3 downsamplers; mid
    ResNet-attention-ResNet at 512; GN + conv_out 512→8; quant_conv 8→8), independently of oracle/.
    A dropped or mis-shaped decoder layer breaks the exact total."""

    def res(ci, co):  # GN, 3×3 conv, GN, 3×3 conv, 1×1 shortcut when the width changes
        return 2 * ci + co * ci * 9 + co + 2 * co + co * co * 9 + co + (co * ci + co if ci != co else 0)

    enc, prev, ch = 3 * 128 * 9 + 128, 128, (128, 256, 512, 512)
    for i, co in enumerate(ch):
        enc += res(prev, co) + res(co, co)
        prev = co
        if i != len(ch) - 1:
            enc += co * co * 9 + co
    enc += 2 * res(512, 512) + 2 * 512 + 4 * (512 * 512 + 512)
    enc += 2 * 512 + 8 * 512 * 9 + 8 + (8 * 8 + 8)
    dec = sum(int(np.prod(s[1])) for s in configs.vae_param_specs(configs.SD_VAE))
    assert enc + dec == 83_653_863


def test_generator_deterministic_and_bounded():
    a = synth.weight(0, "conv_in.weight", (32, 4, 3, 3), synth.KIND_UNIFORM_FANIN, 36)
    b = synth.weight(0, "conv_in.weight", (32, 4, 3, 3), synth.KIND_UNIFORM_FANIN, 36)
    np.testing.assert_array_equal(a, b)
    assert np.abs(a).max() <= 1 / 6 and np.abs(a).max() > 0.15
    assert abs(a.mean()) < 0.02
    c = synth.weight(1, "conv_in.weight", (32, 4, 3, 3), synth.KIND_UNIFORM_FANIN, 36)
    assert not np.array_equal(a, c)
    n = synth.normal(5, 200000)
    assert abs(n.mean()) < 0.01 and abs(n.std() - 1) < 0.01


def test_bf16_round():
    x = np.array([1.0, 1.00390625, 1.005859375, -3.0e-3, 65504.0], dtype=np.float32)
    r = synth.bf16_round(x)
    # 1 + 2^-8 is a tie between 1 and 1+2^-7 → even (1.0); 1.005859375 = 1+3·2^-9 rounds up
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == np.float32(1.0078125)
    assert np.all(np.abs(r - x) <= np.abs(x) * 2.0 ** -8)


def _ctx(n, seed=3):
    return np.stack([synth.text_embedding(seed, i, T.ctx_len, T.ctx_dim) for i in range(n)]).astype(np.float64)


def test_unet_row_independence_and_permutation(P64):
    """I1: each row's ε depends only on its own (x, t, ctx); rows permute with the batch."""
    rng = np.random.default_rng(0)
    x = rng.standard_normal((3, 4, 8, 8))
    t = np.array([951, 501, 1])
    ctx = _ctx(3)
    e = unet.forward(P64, T, x, t, ctx)
    assert e.shape == (3, 4, 8, 8)
    for i in range(3):
        ei = unet.forward(P64, T, x[i:i + 1], t[i:i + 1], ctx[i:i + 1])
        np.testing.assert_allclose(ei[0], e[i], rtol=1e-12, atol=1e-13)
    perm = [2, 0, 1]
    ep = unet.forward(P64, T, x[perm], t[perm], ctx[perm])
    np.testing.assert_allclose(ep, e[perm], rtol=1e-12, atol=1e-13)
    # and the output actually depends on t and ctx (gross-error guard)
    e2 = unet.forward(P64, T, x[:1], np.array([11]), ctx[:1])
    assert np.linalg.norm(e2[0] - e[0]) > 1e-3 * np.linalg.norm(e[0])


def test_unet_fp32_vs_fp64(P64):
    """I2 (R21): fp32 oracle agrees with fp64 to ≤ 1e-5 rel-L2 per step."""
    P32 = configs.unet_params(T, 0, np.float32)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, 4, 8, 8))
    t = np.array([751, 251])
    ctx = _ctx(2)
    e64 = unet.forward(P64, T, x, t, ctx)
    e32 = unet.forward(P32, T, x.astype(np.float32), t, ctx.astype(np.float32))
    assert np.linalg.norm(e32 - e64) / np.linalg.norm(e64) < 1e-5


def test_ddim_closed_forms():
    """I7: ε ≡ 0 telescopes to √(ᾱ_final/ᾱ_t0); ε ≡ e preserves x = √ᾱ x0 + √(1−ᾱ) e."""
    ac = sampling.alphas_cumprod()
    beta = np.linspace(0.00085 ** 0.5, 0.012 ** 0.5, 1000) ** 2
    assert ac[999] == pytest.approx(np.prod(1 - beta), rel=1e-14)
    assert list(sampling.timesteps(4)) == [751, 501, 251, 1]
    assert sampling.timesteps(50)[0] == 981 and sampling.timesteps(50)[-1] == 1
    x = np.ones(5)
    for i in range(50):
        x = sampling.ddim_step(x, np.zeros(5), 50, i)
    np.testing.assert_allclose(x, np.sqrt(ac[0] / ac[981]), rtol=1e-12)
    assert x[0] == pytest.approx(13.1528706, abs=1e-6)
    rng = np.random.default_rng(2)
    x0, e = rng.standard_normal(7), rng.standard_normal(7)
    x = np.sqrt(ac[981]) * x0 + np.sqrt(1 - ac[981]) * e
    for i in range(50):
        x = sampling.ddim_step(x, e, 50, i)
    np.testing.assert_allclose(x, np.sqrt(ac[0]) * x0 + np.sqrt(1 - ac[0]) * e, rtol=1e-12, atol=1e-13)


def test_euler_closed_forms():
    s = sampling.euler_sigmas(20)
    x = np.full(3, 2.0)
    for i in range(20):
        x = sampling.euler_step(x, np.full(3, 0.7), 20, i)
    np.testing.assert_allclose(x, 2.0 - s[0] * 0.7, rtol=1e-13)
    y = np.full(3, 2.0)
    for i in range(20):
        y = sampling.euler_step(y, np.zeros(3), 20, i)
    np.testing.assert_array_equal(y, 2.0)
    assert sampling.init_sigma("euler", 20) == pytest.approx(np.sqrt(s[0] ** 2 + 1))


def test_cfg_pipeline_invariants(P64):
    """I3: g = 1 ≡ cond-only; g = 0 ≡ uncond-only. I4: skipped rows ≡ cond-only."""
    ctx_u = synth.uncond_embedding(0, T.ctx_len, T.ctx_dim).astype(np.float64)
    xT = synth.initial_noise(1, 0, 8, 8).astype(np.float64)
    ctx = _ctx(1)[0]
    a = pipeline.denoise(P64, T, xT, ctx, ctx_u, 4, 1.0, "ddim", skip=set())
    b = pipeline.denoise(P64, T, xT, ctx, ctx_u, 4, 1.0, "ddim", skip=set(range(4)))
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)
    c = pipeline.denoise(P64, T, xT, ctx, ctx_u, 4, 0.0, "ddim", skip=set())
    d = pipeline.denoise(P64, T, xT, ctx_u, ctx_u, 4, 7.5, "ddim", skip=set(range(4)))
    np.testing.assert_allclose(c, d, rtol=1e-12, atol=1e-12)
    e = pipeline.denoise(P64, T, xT, ctx, ctx_u, 4, 7.5, "ddim", skip=set())
    assert np.linalg.norm(e - a) > 1e-3 * np.linalg.norm(a)


def test_step_batch_equals_alone(P64):
    """I5: one ragged step over a batch equals each request stepped alone."""
    ctx_u = synth.uncond_embedding(0, T.ctx_len, T.ctx_dim).astype(np.float64)
    reqs = []
    for i, (n, s, hu, g) in enumerate([(4, 0, True, 7.5), (6, 3, False, 5.0), (4, 2, True, 2.0)]):
        reqs.append(dict(x=synth.initial_noise(1, i, 8, 8).astype(np.float64), ctx=_ctx(3, 9)[i], step=s,
                         n_steps=n, has_uncond=hu, g=g))
    out = pipeline.step_batch(P64, T, reqs, ctx_u, "ddim")
    for i, r in enumerate(reqs):
        alone = pipeline.step_batch(P64, T, [r], ctx_u, "ddim")
        np.testing.assert_allclose(out[i], alone[0], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("c,nb", [(1, 1), (2, 4), (3, 2), (5, 16)])
def test_vae_chunked_equals_whole(V64, c, nb):
    """I6: V1 chunked decode equals the whole decode for any c / band count."""
    z = synth.initial_noise(2, 0, 8, 8).astype(np.float64)[None]
    whole = vae.decode(V64, TV, z)
    assert whole.shape == (1, 3, 16, 16)
    ch = vae.decode_chunked(V64, TV, z, n_chunks=c, n_bands=nb)
    np.testing.assert_allclose(ch, whole, rtol=1e-12, atol=1e-12)


def test_vae_halo0_negative_control(V64):
    z = synth.initial_noise(2, 0, 8, 8).astype(np.float64)[None]
    whole = vae.decode(V64, TV, z)
    bad = vae.decode_chunked(V64, TV, z, n_chunks=2, n_bands=4, halo=0)
    assert np.linalg.norm(bad - whole) / np.linalg.norm(whole) > 1e-3


def test_vae_tiled_v2_reductions_and_error(V64):
    """V2 independent tiles (R7 V2). Pins: (1) a tile covering the image, or a
    halo covering it, reduces to the whole decode exactly (each window IS the whole latent); (2) the
    tile windows partition the latent (every latent pixel owned once, windows clipped at borders);
    (3) it is an approximation — tile-local GroupNorm / attention — so with a small halo it differs
    from the whole decode, and widening the halo brings it closer (the error-vs-halo curve)."""
    z = synth.initial_noise(2, 0, 16, 16).astype(np.float64)[None]
    whole = vae.decode(V64, TV, z)
    np.testing.assert_allclose(vae.decode_tiled(V64, TV, z, tile=16, halo=0), whole, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(vae.decode_tiled(V64, TV, z, tile=8, halo=16), whole, rtol=1e-12, atol=1e-12)
    owned = np.zeros((16, 16), int)
    for (y0, y1, x0, x1), (a0, a1, b0, b1) in vae.tile_windows(16, 16, 8, 4):
        owned[y0:y1, x0:x1] += 1
        assert 0 <= a0 <= y0 < y1 <= a1 <= 16 and 0 <= b0 <= x0 < x1 <= b1 <= 16
    assert (owned == 1).all()
    err = [np.linalg.norm(vae.decode_tiled(V64, TV, z, tile=8, halo=h) - whole) / np.linalg.norm(whole)
           for h in (0, 4, 8)]
    assert err[0] > 1e-3 and err[2] < err[0] and err[2] == 0.0   # halo 8 ≥ image − tile: exact


def _all_partitions(n, c):
    from itertools import combinations
    for cuts in combinations(range(1, n), c - 1):
        yield [0, *cuts, n]


def test_chunk_ranges_minmax(rng):
    for _ in range(200):
        n = int(rng.integers(1, 9))
        c = int(rng.integers(1, 5))
        costs = [int(v) for v in rng.integers(1, 20, n)]
        b = vae.chunk_ranges(costs, c)
        cc = min(c, n)
        assert len(b) == cc + 1 and b[0] == 0 and b[-1] == n and all(b[i] < b[i + 1] for i in range(cc))
        mx = max(sum(costs[b[i]:b[i + 1]]) for i in range(cc))
        opts = [(max(sum(costs[p[i]:p[i + 1]]) for i in range(cc)), p) for p in _all_partitions(n, cc)]
        best = min(o[0] for o in opts)
        assert mx == best
        # ties cut earlier: lexicographically smallest optimal boundary vector
        assert b == min(p for v, p in opts if v == best)


def test_sdxl_param_count():
    # diffusers SDXL-base UNet2DConditionModel has 2,567,463,684 parameters (public count): pins the
    # depth (0, 2, 10) / mid 10 transformers, head-dim heads, linear projections and the 2816-wide
    # "text_time" added embedding of configs.SDXL_UNET
    n = sum(int(np.prod(s[1])) for s in configs.unet_param_specs(configs.SDXL_UNET))
    assert n == 2_567_463_684


def test_generalised_path_reduces_to_sd15_path(P64):
    """The SDXL generalisations with depth 1, linear projections (same values as a 1×1 conv: the
    generator is indexed in canonical layout) and no added embedding are the SD-1.5 network."""
    import dataclasses
    T2 = dataclasses.replace(T, name="tiny_lin", linear_proj=True, tf_depth=(1, 1), mid_depth=1)
    P2 = configs.unet_params(T2, 0, np.float64)
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, 4, 8, 8))
    t = np.array([801, 41])
    ctx = _ctx(2)
    np.testing.assert_allclose(unet.forward(P2, T2, x, t, ctx), unet.forward(P64, T, x, t, ctx), rtol=1e-10,
                               atol=1e-12)


def _xl_inputs(n, seed=7):
    X = configs.TINY_XL_UNET
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, 4, 8, 8))
    ctx = np.stack([synth.text_embedding(seed, i, X.ctx_len, X.ctx_dim) for i in range(n)]).astype(np.float64)
    pooled = np.stack([synth.pooled_embedding(seed, i, X.pooled_dim) for i in range(n)]).astype(np.float64)
    return x, ctx, pooled


def test_tinyxl_rows_depth_and_added_conditioning():
    """I1 for the SDXL-shaped path; the output depends on the pooled embedding and on the time ids
    (added conditioning reaches every ResBlock through temb), and fp32 agrees with fp64 (I2)."""
    X = configs.TINY_XL_UNET
    P = configs.unet_params(X, 0, np.float64)
    x, ctx, pooled = _xl_inputs(3)
    t = np.array([901, 401, 21])
    e = unet.forward(P, X, x, t, ctx, pooled)
    for i in range(3):
        ei = unet.forward(P, X, x[i:i + 1], t[i:i + 1], ctx[i:i + 1], pooled[i:i + 1])
        np.testing.assert_allclose(ei[0], e[i], rtol=1e-12, atol=1e-13)
    e_p = unet.forward(P, X, x[:1], t[:1], ctx[:1], pooled[1:2])
    assert np.linalg.norm(e_p[0] - e[0]) > 1e-4 * np.linalg.norm(e[0])
    ids = np.array([[512, 512, 0, 0, 512, 512]], dtype=np.float64)
    e_t = unet.forward(P, X, x[:1], t[:1], ctx[:1], pooled[:1], ids)
    assert np.linalg.norm(e_t[0] - e[0]) > 1e-4 * np.linalg.norm(e[0])
    P32 = configs.unet_params(X, 0, np.float32)
    e32 = unet.forward(P32, X, x.astype(np.float32), t, ctx.astype(np.float32), pooled.astype(np.float32))
    assert np.linalg.norm(e32 - e) / np.linalg.norm(e) < 1e-5

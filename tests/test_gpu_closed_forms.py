"""SURVEY §8(c) I7 closed forms through the GPU's K12 combine + sampler kernel (sd_debug_combine_update,
an injected ε), i.e. pinned to the mathematics rather than to the oracle:

  DDIM (R4), ε ≡ 0:  x_final = x_T·√(ᾱ_final/ᾱ_{t0}) — the telescoping product; 13.1528706 at n = 50
  DDIM, x_T = √ᾱ_{t0}·x₀ + √(1−ᾱ_{t0})·e and ε ≡ e:  x_final = √ᾱ_final·x₀ + √(1−ᾱ_final)·e
  Euler (R5), ε ≡ κ:  x_final = x_init − σ₀·κ;  ε ≡ 0: x stays constant
  CFG combine (R2/R3): ε_c = ε_u = e gives ε̃ = e for any g; ε_u = 0 gives ε̃ = g·ε_c; a Skip-CFG
  request (no uncond row) uses ε_c whatever the other rows hold.
The kernel computes in fp32 (x ← a·x + b·ε̃ with host-fp64 coefficients), so the bound is a few
hundred fp32 ulps over 50 steps: 2e-5 relative."""
import numpy as np
import pytest
import torch

import synth
from oracle import sampling

pytestmark = pytest.mark.gpu

from paper_2605_08835_b200.engine import Engine  # noqa: E402

TOL = 2e-5


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def engines():
    ed = Engine("tiny", max_latent_hw=16, b_max=4)
    ee = Engine("tiny", max_latent_hw=16, b_max=4, sampler="euler")
    yield ed, ee
    ed.close()
    ee.close()


def _run(eng, xs, n, eps_fn, has_uncond, g):
    lat = [torch.from_numpy(x.copy()).cuda() for x in xs]
    for s in range(n):
        eps = eps_fn(s)
        eng.combine_update(lat, [s] * len(lat), [n] * len(lat), has_uncond, g, torch.from_numpy(eps).cuda())
    return [t.cpu().numpy() for t in lat]


def test_ddim_eps_zero_telescoping(engines):
    ed, _ = engines
    n = 50
    xT = [synth.initial_noise(31, i, 16, 16) for i in range(2)]
    zero = np.zeros((2, 4, 16, 16), np.float32)
    out = _run(ed, xT, n, lambda s: zero, [0, 0], [7.5, 7.5])
    a0, _ = sampling.ddim_alphas(n, 0)
    _, af = sampling.ddim_alphas(n, n - 1)
    factor = np.sqrt(af / a0)
    assert factor == pytest.approx(13.1528706, abs=1e-6)
    for i in range(2):
        assert rel(out[i], factor * xT[i].astype(np.float64)) <= TOL


def test_ddim_form_preservation(engines):
    ed, _ = engines
    n = 20
    x0 = synth.initial_noise(32, 0, 16, 16).astype(np.float64)
    e = synth.initial_noise(32, 1, 16, 16).astype(np.float64)
    a0, _ = sampling.ddim_alphas(n, 0)
    _, af = sampling.ddim_alphas(n, n - 1)
    xT = (np.sqrt(a0) * x0 + np.sqrt(1 - a0) * e).astype(np.float32)
    ef = e.astype(np.float32)[None]
    out = _run(ed, [xT], n, lambda s: ef, [0], [7.5])[0]
    exp = np.sqrt(af) * x0 + np.sqrt(1 - af) * e
    assert rel(out, exp) <= TOL


def test_euler_constant_eps(engines):
    _, ee = engines
    n = 30
    kappa = np.float32(0.37)
    x_init = synth.initial_noise(33, 0, 16, 16) * np.float32(sampling.init_sigma("euler", n))
    const = np.full((1, 4, 16, 16), kappa, np.float32)
    out = _run(ee, [x_init], n, lambda s: const, [0], [7.5])[0]
    s0 = sampling.euler_sigmas(n)[0]
    assert rel(out, x_init.astype(np.float64) - s0 * float(kappa)) <= TOL
    same = _run(ee, [x_init], n, lambda s: np.zeros_like(const), [0], [7.5])[0]
    assert np.array_equal(same, x_init)


def test_cfg_combine_closed_forms(engines):
    ed, _ = engines
    n, s = 10, 3
    a, ap = sampling.ddim_alphas(n, s)
    A = np.sqrt(ap / a)
    Bc = np.sqrt(1 - ap) - np.sqrt(ap * (1 - a) / a)
    x = [synth.initial_noise(34, i, 8, 8) for i in range(3)]
    e = [synth.initial_noise(35, i, 8, 8) for i in range(3)]
    # rows (R26): cond 0, cond 1, cond 2, uncond 0, uncond 1; request 2 skips CFG this step
    g = [7.5, 3.0, 9.0]
    eps = np.stack([e[0], e[1], e[2], e[0], np.zeros_like(e[1])])
    lat = [torch.from_numpy(v.copy()).cuda() for v in x]
    ed.combine_update(lat, [s] * 3, [n] * 3, [1, 1, 0], g, torch.from_numpy(eps).cuda())
    got = [t.cpu().numpy() for t in lat]
    exp = [A * x[0] + Bc * e[0],                 # ε_c = ε_u = e → ε̃ = e for any g
           A * x[1] + Bc * g[1] * e[1],          # ε_u = 0 → ε̃ = g·ε_c
           A * x[2] + Bc * e[2]]                 # Skip-CFG → ε̃ = ε_c
    for i in range(3):
        assert rel(got[i], exp[i]) <= TOL, i

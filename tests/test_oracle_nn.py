"""Pins for oracle/nn.py against brute force, library special cases and closed forms (task ③).

torch fp64 is used here ONLY as an independent library reference (test-only)."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import nn


def _brute_conv(x, w, b, stride, pad):
    N, C, H, W = x.shape
    O, _, kh, kw = w.shape
    Ho = (H + 2 * pad - kh) // stride + 1
    Wo = (W + 2 * pad - kw) // stride + 1
    y = np.zeros((N, O, Ho, Wo))
    for n in range(N):
        for o in range(O):
            for i in range(Ho):
                for j in range(Wo):
                    s = b[o]
                    for c in range(C):
                        for u in range(kh):
                            for v in range(kw):
                                yy, xx = stride * i + u - pad, stride * j + v - pad
                                if 0 <= yy < H and 0 <= xx < W:
                                    s += w[o, c, u, v] * x[n, c, yy, xx]
                    y[n, o, i, j] = s
    return y


@pytest.mark.parametrize("stride,pad,k", [(1, 1, 3), (2, 1, 3), (1, 0, 1)])
def test_conv_bruteforce(rng, stride, pad, k):
    x = rng.standard_normal((2, 3, 6, 5))
    w = rng.standard_normal((4, 3, k, k))
    b = rng.standard_normal(4)
    y = nn.conv2d(x, w, b, stride=stride, pad=pad)
    np.testing.assert_allclose(y, _brute_conv(x, w, b, stride, pad), rtol=1e-12, atol=1e-12)


def test_conv_vs_torch(rng):
    x = rng.standard_normal((2, 16, 9, 7))
    w = rng.standard_normal((8, 16, 3, 3))
    b = rng.standard_normal(8)
    ref = F.conv2d(torch.from_numpy(x), torch.from_numpy(w), torch.from_numpy(b), padding=1).numpy()
    np.testing.assert_allclose(nn.conv2d(x, w, b), ref, rtol=1e-11, atol=1e-11)
    ref2 = F.conv2d(torch.from_numpy(x), torch.from_numpy(w), torch.from_numpy(b), stride=2, padding=1).numpy()
    np.testing.assert_allclose(nn.conv2d(x, w, b, stride=2, pad=1), ref2, rtol=1e-11, atol=1e-11)


def test_groupnorm_definition(rng):
    x = rng.standard_normal((2, 8, 5, 5)) * 3 + 1.5
    y = nn.group_norm(x, 4, np.ones(8), np.zeros(8), 0.0)
    g = y.reshape(2, 4, -1)
    np.testing.assert_allclose(g.mean(axis=2), 0, atol=1e-12)
    np.testing.assert_allclose(g.var(axis=2), 1, atol=1e-12)
    gam, bet = rng.standard_normal(8), rng.standard_normal(8)
    ref = F.group_norm(torch.from_numpy(x), 4, torch.from_numpy(gam), torch.from_numpy(bet), 1e-5).numpy()
    np.testing.assert_allclose(nn.group_norm(x, 4, gam, bet, 1e-5), ref, rtol=1e-11, atol=1e-11)


def test_layernorm(rng):
    x = rng.standard_normal((3, 7, 12)) * 2 - 1
    gam, bet = rng.standard_normal(12), rng.standard_normal(12)
    ref = F.layer_norm(torch.from_numpy(x), (12,), torch.from_numpy(gam), torch.from_numpy(bet), 1e-5).numpy()
    np.testing.assert_allclose(nn.layer_norm(x, gam, bet, 1e-5), ref, rtol=1e-11, atol=1e-11)


def test_attention_properties(rng):
    q = rng.standard_normal((2, 5, 4))
    v = rng.standard_normal((2, 6, 3))
    k_same = np.repeat(rng.standard_normal((2, 1, 4)), 6, axis=1)
    np.testing.assert_allclose(nn.attention(q, k_same, v), np.repeat(v.mean(axis=1, keepdims=True), 5, axis=1),
                               atol=1e-12)
    one = nn.attention(q, rng.standard_normal((2, 1, 4)), v[:, :1])
    np.testing.assert_allclose(one, np.repeat(v[:, :1], 5, axis=1), atol=1e-12)
    k = rng.standard_normal((2, 6, 4))
    eye = np.broadcast_to(np.eye(6), (2, 6, 6)).copy()
    p = nn.attention(q, k, eye)                            # V = I returns the probabilities
    np.testing.assert_allclose(p.sum(axis=-1), 1, atol=1e-12)
    ref = F.scaled_dot_product_attention(torch.from_numpy(q), torch.from_numpy(k), torch.from_numpy(v)).numpy()
    np.testing.assert_allclose(nn.attention(q, k, v), ref, rtol=1e-11, atol=1e-11)


def test_timestep_embedding_closed_form():
    e = nn.timestep_embedding(np.array([0.0, 7.0]), 320, np.float64)
    np.testing.assert_array_equal(e[0, :160], 1.0)
    np.testing.assert_array_equal(e[0, 160:], 0.0)
    # k = 0 frequency is 1: cos(t), sin(t); k = 80: 10000^(-1/2) = 0.01
    assert e[1, 0] == pytest.approx(math.cos(7.0), abs=1e-15)
    assert e[1, 160] == pytest.approx(math.sin(7.0), abs=1e-15)
    assert e[1, 80] == pytest.approx(math.cos(7.0 * 0.01), abs=1e-14)


def test_gelu_silu():
    x = np.linspace(-5, 5, 41)
    ref = np.array([0.5 * t * (1 + math.erf(t / math.sqrt(2))) for t in x])
    np.testing.assert_allclose(nn.gelu(x), ref, rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(nn.silu(x), x / (1 + np.exp(-x)), rtol=1e-15)


def test_silu_closed_values():
    """SiLU(x) = x·σ(x) (R30) pinned by values and identities that do not restate the formula:
    σ(0) = 1/2 ⇒ SiLU(0) = 0 and SiLU'(0) = 1/2; σ(ln 3) = 3/4 ⇒ SiLU(ln 3) = (3/4)·ln 3 and
    SiLU(−ln 3) = −(1/4)·ln 3; σ(x) + σ(−x) = 1 ⇒ SiLU(x) − SiLU(−x) = x; SiLU(x) → x (x → +∞) and
    → 0 (x → −∞); the minimum satisfies x* = −1 − W(1/e), where SiLU(x*) = x* + 1 = −W(1/e)
    = −0.2784645427610738 (Lambert W; omega-constant relation W(1/e)·e^{W(1/e)} = 1/e)."""
    ln3 = math.log(3.0)
    assert nn.silu(np.array([0.0]))[0] == 0.0
    assert nn.silu(np.array([ln3]))[0] == pytest.approx(0.75 * ln3, rel=1e-15)
    assert nn.silu(np.array([-ln3]))[0] == pytest.approx(-0.25 * ln3, rel=1e-15)
    x = np.linspace(-8, 8, 65)
    np.testing.assert_allclose(nn.silu(x) - nn.silu(-x), x, atol=1e-14)
    assert nn.silu(np.array([40.0]))[0] == pytest.approx(40.0, rel=1e-15)
    assert abs(nn.silu(np.array([-40.0]))[0]) < 1e-15
    h = 1e-6
    assert (nn.silu(np.array([h]))[0] - nn.silu(np.array([-h]))[0]) / (2 * h) == pytest.approx(0.5, rel=1e-9)
    g = np.linspace(-1.4, -1.2, 200001)
    assert nn.silu(g).min() == pytest.approx(-0.2784645427610738, abs=1e-12)


def test_upsample():
    x = np.arange(4.0).reshape(1, 1, 2, 2)
    np.testing.assert_array_equal(nn.upsample_nearest2x(x)[0, 0],
                                  [[0, 0, 1, 1], [0, 0, 1, 1], [2, 2, 3, 3], [2, 2, 3, 3]])

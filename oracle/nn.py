"""Plain NumPy layer definitions (ORACLE — test infrastructure only).

NCHW, computed in the dtype of the inputs (fp32 for GPU parity, fp64 for invariants).
Each function is the textbook definition; the conventions the paper leaves open are
SURVEY.md §8(c) R27-R30. Pins: tests/test_oracle_nn.py.
"""
from __future__ import annotations

import numpy as np
from scipy.special import erf


def conv2d(x, w, b=None, stride=1, pad=None):
    """y[n,o,i,j] = b[o] + Σ_{c,u,v} w[o,c,u,v] · xpad[n,c,stride·i+u,stride·j+v]   (im2col + matmul)."""
    N, C, H, W = x.shape
    O, Ci, kh, kw = w.shape
    assert Ci == C, (Ci, C)
    if pad is None:
        pad = kh // 2
    Ho = (H + 2 * pad - kh) // stride + 1
    Wo = (W + 2 * pad - kw) // stride + 1
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad))) if pad else x
    wm = w.reshape(O, C * kh * kw)
    y = np.empty((N, O, Ho, Wo), dtype=np.result_type(x, w))
    for n in range(N):
        cols = np.empty((C, kh, kw, Ho, Wo), dtype=x.dtype)
        for u in range(kh):
            for v in range(kw):
                cols[:, u, v] = xp[n, :, u:u + stride * (Ho - 1) + 1:stride, v:v + stride * (Wo - 1) + 1:stride]
        y[n] = (wm @ cols.reshape(C * kh * kw, Ho * Wo)).reshape(O, Ho, Wo)
    if b is not None:
        y += b.reshape(1, O, 1, 1)
    return y


def linear(x, w, b=None):
    """y = x · wᵀ + b  (w is [out][in], PyTorch layout)."""
    y = x @ w.T
    if b is not None:
        y = y + b
    return y


def group_norm(x, groups, gamma, beta, eps):
    """Two-pass GroupNorm: biased variance, eps inside the sqrt (R29)."""
    N, C = x.shape[:2]
    xg = x.reshape(N, groups, -1)
    mean = xg.mean(axis=2, keepdims=True)
    var = ((xg - mean) ** 2).mean(axis=2, keepdims=True)
    y = ((xg - mean) / np.sqrt(var + eps)).reshape(x.shape)
    shp = (1, C) + (1,) * (x.ndim - 2)
    return y * gamma.reshape(shp) + beta.reshape(shp)


def layer_norm(x, gamma, beta, eps):
    mean = x.mean(axis=-1, keepdims=True)
    var = ((x - mean) ** 2).mean(axis=-1, keepdims=True)
    return (x - mean) / np.sqrt(var + eps) * gamma + beta


def silu(x):
    return x / (1.0 + np.exp(-x))


def gelu(x):
    """Exact (erf) GELU (R30)."""
    return 0.5 * x * (1.0 + erf(x / np.sqrt(2.0)).astype(x.dtype))


def softmax(s, axis=-1):
    m = s.max(axis=axis, keepdims=True)
    e = np.exp(s - m)
    return e / e.sum(axis=axis, keepdims=True)


def attention(q, k, v):
    """softmax(q kᵀ / √d) v per head. q [..., L, d], k/v [..., S, d] (R28)."""
    d = q.shape[-1]
    scale = 1.0 / np.sqrt(d)
    out = np.empty(q.shape[:-1] + (v.shape[-1],), dtype=q.dtype)
    lead = q.shape[:-2]
    for idx in np.ndindex(*lead):
        s = (q[idx] @ k[idx].T) * q.dtype.type(scale)
        out[idx] = softmax(s) @ v[idx]
    return out


def upsample_nearest2x(x):
    return x.repeat(2, axis=2).repeat(2, axis=3)


def timestep_embedding(t, dim, dtype=np.float32, max_period=10000.0):
    """Sinusoid, flip_sin_to_cos=True, shift 0 (R27): [cos(t·f) ‖ sin(t·f)], f_k = exp(-ln(P)·k/half)."""
    half = dim // 2
    k = np.arange(half, dtype=np.float64)
    freqs = np.exp(-np.log(max_period) * k / half).astype(dtype)
    args = np.asarray(t, dtype=dtype).reshape(-1, 1) * freqs.reshape(1, -1)
    return np.concatenate([np.cos(args), np.sin(args)], axis=1).astype(dtype)

"""Seeded synthetic-input generators shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no convolution, attention,
sampler, CFG or scheduling math). It only turns (seed, name, index) into
numbers, so that the oracle (`oracle/`) and the product path
(`paper_2605_08835_b200/`) can be fed identical inputs without importing each
other (task rule ③).

Generator (re-specified as a counter-based generator so
that the CUDA weight-init kernel can implement the same function on device):

  tensor_seed(global_seed, name) = mix64(fnv1a64(name) ^ mix64(global_seed))
  bits_i                         = mix64(tensor_seed + (i + 1) * 0x9E3779B97F4A7C15)   (mod 2^64)
  u_i   = (bits_i >> 40) * 2^-24                       exactly representable fp32 in [0, 1)
  t_i   = (u_i - 0.5) * 2                               exact in fp32
  uniform(±b)_i = fl32(t_i * b), b = fl32(bound)        one IEEE fp32 multiply

mix64 is the SplitMix64 finaliser. The CUDA side (csrc/weights.cu) implements
the same function; `index` is the element's flat index in the canonical
(PyTorch/diffusers) layout of the tensor: conv [O][I][kh][kw], linear [O][I].

Normals (text embeddings, initial noise) are Box-Muller in fp64 over two
counters (2i, 2i+1) and rounded to fp32; the C++ serving path implements the
same formula with libm.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_FNV_OFF = 0xCBF29CE484222325
_FNV_PRIME = 0x100000001B3
_MASK = (1 << 64) - 1


def mix64_int(z: int) -> int:
    """SplitMix64 finaliser on a Python int (mod 2^64)."""
    z &= _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


def _mix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def fnv1a64(s: str) -> int:
    h = _FNV_OFF
    for b in s.encode("utf-8"):
        h ^= b
        h = (h * _FNV_PRIME) & _MASK
    return h


def tensor_seed(global_seed: int, name: str) -> int:
    return mix64_int(fnv1a64(name) ^ mix64_int(int(global_seed)))


def _bits(seed: int, start: int, n: int) -> np.ndarray:
    idx = np.arange(start + 1, start + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + idx * GOLDEN
    return _mix64(z)


def unit_uniform(seed: int, n: int, start: int = 0) -> np.ndarray:
    """u_i in [0,1), fp32, 24-bit resolution (exact)."""
    b = _bits(seed, start, n) >> np.uint64(40)
    return (b.astype(np.float32) * np.float32(2.0 ** -24)).astype(np.float32)


def uniform_pm(seed: int, n: int, bound: float) -> np.ndarray:
    """U(-bound, bound) as fl32((u-0.5)*2 * fl32(bound))."""
    u = unit_uniform(seed, n)
    t = (u - np.float32(0.5)) * np.float32(2.0)
    return (t * np.float32(bound)).astype(np.float32)


def normal(seed: int, n: int) -> np.ndarray:
    """Box-Muller N(0,1) in fp64 → fp32. Uses counters 2i and 2i+1."""
    b = _bits(seed, 0, 2 * n)
    u = (b >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    u1 = 1.0 - u[0::2]          # (0, 1]
    u2 = u[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    return (r * np.cos(2.0 * np.pi * u2)).astype(np.float32)


# ---- weight kinds (R20) ---------------------------------------------------------------------
KIND_UNIFORM_FANIN = 0   # U(±1/sqrt(fan_in))   weights and biases
KIND_NORM_GAMMA = 1      # 1 + U(±0.1)
KIND_NORM_BETA = 2       # U(±0.1)


def weight(global_seed: int, name: str, shape, kind: int, fan_in: int = 1, gain: float = 1.0) -> np.ndarray:
    """One parameter tensor in canonical (PyTorch) layout, fp32."""
    n = int(np.prod(shape))
    seed = tensor_seed(global_seed, name)
    if kind == KIND_UNIFORM_FANIN:
        bound = np.float32(np.float32(1.0 / np.sqrt(float(fan_in))) * np.float32(gain))
        v = uniform_pm(seed, n, float(bound))
    elif kind == KIND_NORM_GAMMA:
        v = (np.float32(1.0) + uniform_pm(seed, n, 0.1)).astype(np.float32)
    elif kind == KIND_NORM_BETA:
        v = uniform_pm(seed, n, 0.1)
    else:
        raise ValueError(kind)
    return v.reshape(shape)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as fp32 (what the GPU stores)."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = (u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)
    out = (r << np.uint64(16)).astype(np.uint32).view(np.float32)
    nan = np.isnan(a)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out.reshape(x.shape)


def text_embedding(trace_seed: int, req_id: int, length: int, dim: int) -> np.ndarray:
    """Synthetic prompt embedding [length][dim] ~ N(0,1) (A14 is OUT; R20)."""
    return normal(tensor_seed(trace_seed, f"ctx/{req_id}"), length * dim).reshape(length, dim)


def uncond_embedding(weight_seed: int, length: int, dim: int) -> np.ndarray:
    """The shared unconditional (empty-prompt) embedding, fixed seed (R20)."""
    return normal(tensor_seed(weight_seed, "ctx/uncond"), length * dim).reshape(length, dim)


def pooled_embedding(trace_seed: int, req_id: int, dim: int) -> np.ndarray:
    """Synthetic pooled text embedding [dim] ~ N(0,1) for SDXL's added conditioning (R20, R27)."""
    return normal(tensor_seed(trace_seed, f"pooled/{req_id}"), dim)


def uncond_pooled(weight_seed: int, dim: int) -> np.ndarray:
    """The unconditional pooled embedding (SDXL), fixed seed (R20)."""
    return normal(tensor_seed(weight_seed, "pooled/uncond"), dim)


def initial_noise(trace_seed: int, req_id: int, h: int, w: int) -> np.ndarray:
    """z ~ N(0,1) [4][h][w] per (trace seed, id) (R20)."""
    return normal(tensor_seed(trace_seed, f"noise/{req_id}"), 4 * h * w).reshape(4, h, w)

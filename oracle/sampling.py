"""Samplers and classifier-free guidance (ORACLE — test infrastructure only).

The paper gives no sampler and no CFG formula (PAPER.md:162
mentions only "the standard CFG mechanism"). Readings:
  R2  ε̃ = ε_u + g·(ε_c − ε_u)
  R3  a skipped step (Skip-CFG) uses ε̃ = ε_c
  R4  DDIM, η = 0, scaled-linear β, "leading" spacing, steps_offset 1, set_alpha_to_one False
  R5  Euler (ε-prediction, no churn) on the same integer grid
Coefficients are computed in fp64 (the GPU host side does the same and passes fp32).
"""
from __future__ import annotations

import numpy as np

N_TRAIN = 1000


def alphas_cumprod():
    beta = np.linspace(np.sqrt(0.00085), np.sqrt(0.012), N_TRAIN, dtype=np.float64) ** 2
    return np.cumprod(1.0 - beta)


def timesteps(n_steps: int):
    """t_i = (n−1−i)·Δ + 1, Δ = 1000 // n (R4 'leading' + steps_offset 1)."""
    d = N_TRAIN // n_steps
    return np.array([(n_steps - 1 - i) * d + 1 for i in range(n_steps)], dtype=np.int64)


def ddim_alphas(n_steps: int, i: int):
    """(ᾱ_t, ᾱ_prev) for step index i."""
    ac = alphas_cumprod()
    d = N_TRAIN // n_steps
    t = int(timesteps(n_steps)[i])
    tp = t - d
    return ac[t], (ac[tp] if tp >= 0 else ac[0])


def ddim_step(x, eps, n_steps: int, i: int):
    """x̂₀ = (x − √(1−ᾱ_t)·ε̃)/√ᾱ_t ;  x ← √ᾱ_prev·x̂₀ + √(1−ᾱ_prev)·ε̃   (η = 0, no clipping)."""
    a, ap = ddim_alphas(n_steps, i)
    dt = x.dtype.type
    x0 = (x - dt(np.sqrt(1.0 - a)) * eps) / dt(np.sqrt(a))
    return dt(np.sqrt(ap)) * x0 + dt(np.sqrt(1.0 - ap)) * eps


def euler_sigmas(n_steps: int):
    ac = alphas_cumprod()
    ts = timesteps(n_steps)
    s = np.sqrt((1.0 - ac[ts]) / ac[ts])
    return np.concatenate([s, [0.0]])


def init_sigma(sampler: str, n_steps: int) -> float:
    if sampler == "ddim":
        return 1.0
    s0 = euler_sigmas(n_steps)[0]
    return float(np.sqrt(s0 * s0 + 1.0))


def c_in(sampler: str, n_steps: int, i: int) -> float:
    if sampler == "ddim":
        return 1.0
    s = euler_sigmas(n_steps)[i]
    return float(1.0 / np.sqrt(s * s + 1.0))


def euler_step(x, eps, n_steps: int, i: int):
    s = euler_sigmas(n_steps)
    return x + x.dtype.type(s[i + 1] - s[i]) * eps


def step(sampler: str, x, eps, n_steps: int, i: int):
    return ddim_step(x, eps, n_steps, i) if sampler == "ddim" else euler_step(x, eps, n_steps, i)


def cfg_combine(eps_c, eps_u, g, has_uncond: bool):
    """R2 / R3."""
    if not has_uncond:
        return eps_c
    return eps_u + eps_c.dtype.type(g) * (eps_c - eps_u)

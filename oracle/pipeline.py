"""One step-level batched denoising iteration and a whole-request loop (ORACLE — test infrastructure only).

`step_batch` is the plain definition of what `sd_step_batch` computes (
PAPER.md:162, :230 for Skip-CFG; R2-R5, R26):
  rows = [cond rows of all requests in batch order] + [uncond rows of requests with has_uncond]
  ε    = UNet(c_in(t_r)·x_r, t_r, ctx_row)
  ε̃_r  = has_uncond_r ? ε_u + g_r(ε_c − ε_u) : ε_c
  x_r ← sampler(x_r, ε̃_r, step s_r)
"""
from __future__ import annotations

import numpy as np

from . import sampling, unet


def step_batch(P, cfg, reqs, ctx_uncond, sampler="ddim", pooled_uncond=None):
    """reqs: list of dict(x [4,h,w], ctx [L,D], step s_r, n_steps n_r, has_uncond, g[, pooled (SDXL)]).
    Returns new x list."""
    if not reqs:
        return []
    dt = reqs[0]["x"].dtype
    rows_x, rows_t, rows_c, rows_p = [], [], [], []
    order = [(i, False) for i in range(len(reqs))] + [(i, True) for i, r in enumerate(reqs) if r["has_uncond"]]
    for i, unc in order:
        r = reqs[i]
        t = int(sampling.timesteps(r["n_steps"])[r["step"]])
        rows_x.append(r["x"] * dt.type(sampling.c_in(sampler, r["n_steps"], r["step"])))
        rows_t.append(t)
        rows_c.append(ctx_uncond if unc else r["ctx"])
        if cfg.add_time_dim:
            rows_p.append(pooled_uncond if unc else r["pooled"])
    pooled = np.stack(rows_p).astype(dt) if cfg.add_time_dim else None
    eps = unet.forward(P, cfg, np.stack(rows_x), np.array(rows_t), np.stack(rows_c).astype(dt), pooled)
    out = []
    uidx = {i: len(reqs) + k for k, i in enumerate([i for i, u in order[len(reqs):]])}
    for i, r in enumerate(reqs):
        ec = eps[i]
        eu = eps[uidx[i]] if r["has_uncond"] else None
        et = sampling.cfg_combine(ec, eu, r["g"], r["has_uncond"])
        out.append(sampling.step(sampler, r["x"], et, r["n_steps"], r["step"]))
    return out


def denoise(P, cfg, x_T, ctx, ctx_uncond, n_steps, g, sampler="ddim", skip=frozenset()):
    """A request run alone: x = init_sigma·x_T, then n steps; step i skips CFG iff i ∈ skip."""
    x = x_T * x_T.dtype.type(sampling.init_sigma(sampler, n_steps))
    for i in range(n_steps):
        x = step_batch(P, cfg, [dict(x=x, ctx=ctx, step=i, n_steps=n_steps, has_uncond=(i not in skip), g=g)],
                       ctx_uncond, sampler)[0]
    return x

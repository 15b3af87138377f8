"""Serving driver: synthetic request traces (PAPER.md:315 workload shape) played against the GPU
server behind sd_serve_start / sd_submit / sd_poll, plus the E2E metrics of PAPER.md:325 (R18).

Traces: Poisson arrivals at rate λ (tasks/s) or a burst (a fraction of the requests inside a short
window, "dispatching 50% of total tasks within a concentrated short interval"); steps
uniform in [20, 50]; one resolution per server (R22); prompt embeddings and noise seeded per id (R20).
Marshalling only — the serving loop, planner, controller and every kernel run in libsynerdiff.so.
"""
from __future__ import annotations

import ctypes as C
import math
import time

import numpy as np

import synth

from . import binding as B


def poisson_trace(n, rate, seed=7, steps=(20, 50), t0_us=0):
    rng = np.random.default_rng(seed)
    gaps = rng.exponential(1e6 / rate, n) if rate > 0 else np.zeros(n)
    arr = t0_us + np.cumsum(gaps) - gaps[0]
    st = rng.integers(steps[0], steps[1] + 1, n)
    return [(i, int(arr[i]), int(st[i])) for i in range(n)]


def burst_trace(n, base_rate, frac=0.5, span_us=10_000_000, seed=7, steps=(20, 50)):
    rng = np.random.default_rng(seed)
    nb = int(round(frac * n))
    rest = poisson_trace(n - nb, base_rate, seed + 1, steps)
    t_mid = rest[len(rest) // 2][1] if rest else 0
    b = sorted(int(t_mid + x) for x in rng.uniform(0, span_us, nb))
    st = rng.integers(steps[0], steps[1] + 1, nb)
    merged = sorted([(a, s) for _, a, s in rest] + list(zip(b, st.tolist())))
    return [(i, a, int(s)) for i, (a, s) in enumerate(merged)]


def p99(values):
    v = sorted(values)
    r = -(-99 * len(v) // 100)
    return v[max(r, 1) - 1]


def run_trace(eng, table_h, trace, latent_hw=64, b_max=8, c_star=1, c_max=2, dp_mode=0, guidance=7.5,
              trace_seed=7, ctl=None, timeout_s=600, n_max=None, policy="synerdiff", ablation=0,
              dyn_window_us=500_000, res_tables=None, trajectory=None, vae_sms=0):
    """Serve `trace` [(id, arrival_us, n_steps[, latent_hw])] on `eng`; returns per-request records and
    metrics. `res_tables` {latent_hw: table handle} makes the server mixed-resolution. A list passed as
    `trajectory` receives the controller trajectory (one dict per planned window, sd_serve_window_log).
    Arrival times are relative to sd_serve_start; all requests are submitted up front and admitted
    by the server when their arrival time has passed. `policy` selects SynerDiff or one of the
    paper's baselines, `ablation` the SD_ABL_* bits. `vae_sms` > 0
    runs the VAE chunks and the UNet rounds on disjoint green-context SM partitions (sd_serve_config)."""
    ctl = ctl or B.ControllerConfig(c_star, c_max, 10, 3, 1, 2, -1, 5)
    cfg = B.ServeConfig(b_max, 1, 10, dp_mode, c_star, ctl, table_h, latent_hw, trace_seed, n_max or 0,
                        B.POLICIES[policy], ablation, dyn_window_us)
    cfg.vae_sms = vae_sms
    if res_tables:
        keys = sorted(res_tables)
        hw_arr = (C.c_int32 * len(keys))(*keys)
        tb_arr = (C.c_void_p * len(keys))(*[res_tables[k].value for k in keys])
        cfg.n_res = len(keys)
        cfg.res_hw = C.cast(hw_arr, C.POINTER(C.c_int32))
        cfg.res_tables = C.cast(tb_arr, C.POINTER(C.c_void_p))
    embs = {e[0]: np.ascontiguousarray(synth.text_embedding(trace_seed, e[0], eng.ctx_len, eng.ctx_dim))
            for e in trace}
    pooled = {e[0]: np.ascontiguousarray(synth.pooled_embedding(trace_seed, e[0], eng.pooled_dim))
              for e in trace} if eng.pooled_dim else {}
    B.call("sd_serve_start", eng.h, C.byref(cfg))
    try:
        for e in trace:
            i, a, n = e[:3]
            r = B.Request(i, a, n, guidance, embs[i].ctypes.data, eng.ctx_len, eng.ctx_dim,
                          pooled[i].ctypes.data if pooled else None, eng.pooled_dim, e[3] if len(e) > 3 else 0)
            B.call("sd_submit", eng.h, C.byref(r))
        out = (B.Completion * 64)()
        cnt = C.c_int32()
        recs = {}
        t_end = time.time() + timeout_s
        while len(recs) < len(trace) and time.time() < t_end:
            B.call("sd_poll", eng.h, out, 64, C.byref(cnt), 100)
            for j in range(cnt.value):
                c = out[j]
                recs[c.id] = dict(A=c.arrival_us, U=c.denoise_done_us, V=c.decode_done_us, skips=c.n_skipped)
                B.call("sd_release", eng.h, c.id)
        if trajectory is not None:
            cap = 1 << 16
            cols = {k: (C.c_int64 * cap)() if k in ("t0", "t1") else (C.c_int32 * cap)()
                    for k in ("t0", "t1", "M", "N", "K", "level", "c", "waiting", "level_after", "c_after")}
            nw = C.c_int32()
            B.call("sd_serve_window_log", eng.h, cap, *cols.values(), C.byref(nw))
            trajectory.extend({k: int(v[i]) for k, v in cols.items()} for i in range(nw.value))
    finally:
        B.call("sd_serve_stop", eng.h)
    if len(recs) < len(trace):
        raise RuntimeError(f"serving timed out: {len(recs)}/{len(trace)} completed")
    e2e = [r["V"] - r["A"] for r in recs.values()]
    span = max(r["V"] for r in recs.values()) - min(r["A"] for r in recs.values())
    metrics = dict(n=len(e2e), images_per_s=len(e2e) / (span / 1e6), mean_e2e_ms=float(np.mean(e2e)) / 1e3,
                   p99_e2e_ms=p99(e2e) / 1e3, skipped_steps=int(sum(r["skips"] for r in recs.values())),
                   denoise_steps=int(sum(e[2] for e in trace)))
    return recs, metrics

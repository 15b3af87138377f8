"""Mixed-resolution serving on one B200 (PAPER.md:315 mixes resolutions): SD-1.5
requests at 512² and 768² (latent 64 / 96, half each) in one Poisson trace, steps U{20..50}, g 7.5,
B_max 8. Per-resolution τ/δ tables (c ∈ {1, 2}) are profiled on the GPU; each window plans with the
table of its largest resolution; each round runs one sd_step_batch per resolution group. SynerDiff
against the baselines, GPU server beside the virtual clock.

  python tools/mixed_sweep.py [--requests 48] [--rho 0.8 1.2] [--out profiles/r01/mixed_sweep.json]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_08835_b200 import binding as B  # noqa: E402
from paper_2605_08835_b200 import profiler, serving  # noqa: E402
from paper_2605_08835_b200.engine import Engine  # noqa: E402

RES = (64, 96)


def simulate(handles, trace, policy, c_star, c_max):
    n = len(trace)
    ctl = B.ControllerConfig(c_star, c_max, 10, 3, 1, 2, -1, 5)
    keys = sorted(handles)
    hw = (C.c_int32 * len(keys))(*keys)
    tb = (C.c_void_p * len(keys))(*[handles[k].value for k in keys])
    cfg = B.ServeConfig(8, 1, 10, 0, c_star, ctl, None, 64, 7, 3, B.POLICIES[policy], 0, 500_000, len(keys),
                        C.cast(hw, C.POINTER(C.c_int32)), C.cast(tb, C.POINTER(C.c_void_p)))
    U, V = (C.c_int64 * n)(), (C.c_int64 * n)()
    ns, win = (C.c_int32 * n)(), C.c_int32()
    B.call("sd_serve_simulate_mixed", C.byref(cfg), n, (C.c_uint64 * n)(*[t[0] for t in trace]),
           (C.c_int64 * n)(*[t[1] for t in trace]), (C.c_int32 * n)(*[t[2] for t in trace]),
           (C.c_int32 * n)(*[t[3] for t in trace]), U, V, ns, C.byref(win))
    e2e = [V[i] - trace[i][1] for i in range(n)]
    span = max(V) - min(t[1] for t in trace)
    return dict(images_per_s=n / (span / 1e6), mean_e2e_ms=sum(e2e) / n / 1e3, p99_e2e_ms=serving.p99(e2e) / 1e3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=48)
    ap.add_argument("--rho", type=float, nargs="+", default=[0.8, 1.2])
    ap.add_argument("--out", default="profiles/r01/mixed_sweep.json")
    args = ap.parse_args()
    eng = Engine("sd15", max_latent_hw=96, b_max=8, c_max=2)
    eng.set_uncond(torch.from_numpy(synth.uncond_embedding(0, 77, 768)))
    handles, tabs = {}, {}
    t0 = time.time()
    for r in RES:
        eng.warmup(r, r, 8, n_dec=3)
        prof = profiler.Profiler(eng, r, r, 8, reps=1)
        tabs[r] = prof.measure([1, 2], b_max=8, n_max=3)
        prof.close()
        handles[r] = profiler.to_table_handle(tabs[r])
    c_max, c_star, _ = profiler.chunk_choice(tabs[96], [1, 2], m=8, n=1)
    c_max = max(c_max, c_star)
    print(f"profiled {RES} in {time.time() - t0:.1f} s; c* = {c_star}, C_max = {c_max}", flush=True)
    rng = np.random.default_rng(5)
    cal = [(i, 0, n, int(rng.choice(RES))) for (i, _, n) in serving.poisson_trace(16, 0.0, seed=11)]
    serving.run_trace(eng, None, cal, 64, 8, c_star, c_max, n_max=3, res_tables=handles)
    _, m = serving.run_trace(eng, None, cal, 64, 8, c_star, c_max, n_max=3, res_tables=handles)
    c1 = m["images_per_s"]
    print(f"C1 (mixed) = {c1:.3f} images/s", flush=True)
    res = dict(workload=f"SD-1.5 mixed 512² / 768² (latent 64 / 96, half each), {args.requests} Poisson requests "
                        "per load, steps U{20..50}, g 7.5, B_max 8, λ = ρ·C₁(mixed)",
               c1_images_per_s=c1, c_star=c_star, c_max=c_max, loads={})
    for rho in args.rho:
        base = serving.poisson_trace(args.requests, rho * c1, seed=7)
        trace = [(i, a, n, int(rng.choice(RES))) for (i, a, n) in base]
        row = {}
        for pol in ("synerdiff", "naive", "dynamic", "serial"):
            cs, cm = (c_star, c_max) if pol == "synerdiff" else (1, 1)
            _, g = serving.run_trace(eng, None, trace, 64, 8, cs, cm, n_max=3, policy=pol, res_tables=handles)
            sim = simulate(handles, trace, pol, cs, cm)
            row[pol] = dict(gpu=g, virtual_clock=sim)
            print(f"rho {rho}: {pol:10s} {g['images_per_s']:.3f} img/s, mean {g['mean_e2e_ms']:.0f} ms, "
                  f"P99 {g['p99_e2e_ms']:.0f} ms, skips {g['skipped_steps']} | sim {sim['images_per_s']:.3f} img/s, "
                  f"mean {sim['mean_e2e_ms']:.0f}, P99 {sim['p99_e2e_ms']:.0f}", flush=True)
        res["loads"][str(rho)] = row
    for h in handles.values():
        B.lib().sd_table_free(h)
    eng.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

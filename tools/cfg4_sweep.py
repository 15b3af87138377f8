"""CFG#4-shaped serving on one B200: SD-1.5 at 768² (latent 96×96) under high load with
the threshold-aware plan and the feedback controller on; per-GPU weak-scaling point λ = ρ·C₁ with
ρ ∈ {0.95, 1.1} (requests shard id mod P across GPUs with no data-path collective, so each of P GPUs
serves this trace). Reports images/s, mean / P99 E2E and the controller trajectory (Skip-CFG level and
chunk count per window, from sd_serve_window_log).

  python tools/cfg4_sweep.py [--requests 64] [--rho 0.95 1.1]
"""
import argparse
import collections
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_08835_b200 import binding as B  # noqa: E402
from paper_2605_08835_b200 import profiler, serving  # noqa: E402
from paper_2605_08835_b200.engine import Engine  # noqa: E402

LAT = 96


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=64)
    ap.add_argument("--rho", type=float, nargs="+", default=[0.95, 1.1])
    ap.add_argument("--out", default="profiles/r01/cfg4_sweep.json")
    args = ap.parse_args()
    eng = Engine("sd15", max_latent_hw=LAT, b_max=8, c_max=3)
    eng.set_uncond(torch.from_numpy(synth.uncond_embedding(0, 77, 768)))
    t0 = time.time()
    eng.warmup(LAT, LAT, 8, n_dec=3)
    prof = profiler.Profiler(eng, LAT, LAT, 8, reps=1)
    cs = [1, 2, 3]  # the controller steps c by one up to C_max: every c in [1, C_max] needs a table
    tab = prof.measure(cs, b_max=8, n_max=3)
    prof.close()
    h = profiler.to_table_handle(tab)
    c_max, c_star, _ = profiler.chunk_choice(tab, cs, m=8, n=1)
    c_max = min(max(c_max, c_star, 2), cs[-1])  # let the controller escalate c at least once
    print(f"profiled {len(tab)} entries in {time.time() - t0:.0f} s; c* = {c_star}, C_max = {c_max}", flush=True)
    cal = [(i, 0, n) for (i, _, n) in serving.poisson_trace(16, 0.0, seed=11)]
    serving.run_trace(eng, h, cal, LAT, 8, c_star, c_max, n_max=3)
    _, m = serving.run_trace(eng, h, cal, LAT, 8, c_star, c_max, n_max=3)
    c1 = m["images_per_s"]
    print(f"C1 = {c1:.3f} images/s", flush=True)
    res = dict(workload=f"SD-1.5 768² (latent 96), {args.requests} Poisson requests per load, steps U{{20..50}}, "
                        f"g 7.5, B_max 8, controller on (c* = {c_star}, C_max = {c_max}), λ = ρ·C₁ per GPU",
               c1_images_per_s=c1, c_star=c_star, c_max=c_max, loads={})
    for rho in args.rho:
        trace = serving.poisson_trace(args.requests, rho * c1, seed=7)
        traj = []
        _, g = serving.run_trace(eng, h, trace, LAT, 8, c_star, c_max, n_max=3, trajectory=traj)
        lv = collections.Counter(w["level"] for w in traj)
        cc = collections.Counter(w["c"] for w in traj)
        changes = sum(1 for w in traj if (w["level_after"], w["c_after"]) != (w["level"], w["c"]))
        summary = dict(windows=len(traj), level_hist=dict(lv), c_hist=dict(cc), changes=changes,
                       max_waiting=max((w["waiting"] for w in traj), default=0))
        res["loads"][str(rho)] = dict(metrics=g, controller=summary, trajectory=traj)
        print(f"rho {rho}: {g['images_per_s']:.3f} img/s, mean {g['mean_e2e_ms']:.0f} ms, P99 {g['p99_e2e_ms']:.0f} ms, "
              f"skips {g['skipped_steps']}; controller {summary}", flush=True)
    B.lib().sd_table_free(h)
    eng.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

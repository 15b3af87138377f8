"""SynerDiff vs the paper's baselines and ablations on one B200 (§IV Baselines,
:352-357 throughput / E2E evaluation, :395-397 ablation).

SD-1.5-shaped UNet + VAE at 512² (latent 64×64), B_max = 8, steps U{20..50}, g = 7.5.
  1. offline profiler → τ/δ table for c ∈ {1, 2} (§III-C) and c*, C_max;
  2. C₁ = SynerDiff's saturation throughput (16 requests at t = 0);
  3. for each load ρ, one Poisson trace at λ = ρ·C₁ served by every policy on the GPU server
     (sd_serve_start / sd_submit / sd_poll): images/s, mean and P99 E2E (R18);
  4. the same traces on the virtual clock (sd_serve_simulate on the measured table) beside them.

  python tools/policy_sweep.py [--requests 48] [--rho 0.5 0.8 1.1 1.5] [--burst] [--out profiles/r01/policy_sweep.json]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_08835_b200 import binding as B  # noqa: E402
from paper_2605_08835_b200 import profiler, serving  # noqa: E402
from paper_2605_08835_b200.engine import Engine  # noqa: E402

# name → (policy, ablation bits, chunking on)
ARMS = {
    "synerdiff": ("synerdiff", 0, True),
    "naive (InstGenIE)": ("naive", 0, False),
    "dynamic batching": ("dynamic", 0, False),
    "serial (Diffusers BS=1)": ("serial", 0, False),
    "synerdiff w/o skip-cfg": ("synerdiff", B.SD_ABL_NO_SKIP, True),
    "synerdiff w/o chunking": ("synerdiff", 0, False),
    "synerdiff w/o controller": ("synerdiff", B.SD_ABL_NO_CTL, True),
}


def simulate(h, trace, policy, ablation, c_star, c_max):
    n = len(trace)
    ctl = B.ControllerConfig(c_star, c_max, 10, 3, 1, 2, -1, 5)
    cfg = B.ServeConfig(8, 1, 10, 0, c_star, ctl, h, 64, 7, 3, B.POLICIES[policy], ablation, 500_000)
    U, V = (C.c_int64 * n)(), (C.c_int64 * n)()
    ns, win = (C.c_int32 * n)(), C.c_int32()
    B.call("sd_serve_simulate", C.byref(cfg), h, n, (C.c_uint64 * n)(*[t[0] for t in trace]),
           (C.c_int64 * n)(*[t[1] for t in trace]), (C.c_int32 * n)(*[t[2] for t in trace]), U, V, ns, C.byref(win))
    e2e = [V[i] - trace[i][1] for i in range(n)]
    span = max(V) - min(t[1] for t in trace)
    return dict(images_per_s=n / (span / 1e6), mean_e2e_ms=sum(e2e) / n / 1e3, p99_e2e_ms=serving.p99(e2e) / 1e3,
                skipped_steps=int(sum(ns)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=48)
    ap.add_argument("--rho", type=float, nargs="+", default=[0.5, 0.8, 1.1, 1.5])
    ap.add_argument("--burst", action="store_true",
                    help="also a burst trace: half the requests inside a window at 2·C₁ on a 0.5·C₁ background "
                         "(PAPER.md:315 burst traffic)")
    ap.add_argument("--arms", nargs="+", default=list(ARMS))
    ap.add_argument("--c1-requests", type=int, default=16,
                    help="requests of the saturation trace (all arriving at t = 0) that defines C1; CFG#3 of "
                         "SURVEY 8(d) uses the full trace size")
    ap.add_argument("--burst-span-s", type=float, default=0.0,
                    help="burst window in seconds (CFG#3 / S:499: 10); 0 = half the requests at 2*C1")
    ap.add_argument("--no-sim", action="store_true", help="skip the virtual-clock replay")
    ap.add_argument("--vae-sms", type=int, nargs="+", default=[0],
                    help="SM partition sizes for the VAE (0 = stream priority only); each arm runs once per value")
    ap.add_argument("--out", default="profiles/r01/policy_sweep.json")
    args = ap.parse_args()
    eng = Engine("sd15", max_latent_hw=64, b_max=8, c_max=2)
    eng.set_uncond(torch.from_numpy(synth.uncond_embedding(0, 77, 768)))
    t0 = time.time()
    eng.warmup(64, 64, 8, n_dec=3)     # every step-shape graph and 3 pooled decode states
    print(f"warm-up {time.time() - t0:.1f} s", flush=True)
    t0 = time.time()
    prof = profiler.Profiler(eng, 64, 64, 8, reps=1)
    tab = prof.measure([1, 2], b_max=8, n_max=3)
    prof.close()
    h = profiler.to_table_handle(tab)
    part_tables = {}  # vae_sms → table profiled on that SM partition (the planner must see its own timings)
    for vs in args.vae_sms:
        if vs > 0:
            pp = profiler.Profiler(eng, 64, 64, 8, reps=1, vae_sms=vs)
            part_tables[vs] = (profiler.to_table_handle(pp.measure([1, 2], b_max=8, n_max=3)), pp.partition_sms)
            pp.close()
            print(f"profiled the {pp.partition_sms} SM partition", flush=True)
    c_max, c_star, _ = profiler.chunk_choice(tab, [1, 2], m=8, n=1)
    c_max = max(c_max, c_star)
    print(f"profiled {len(tab)} table entries in {time.time() - t0:.1f} s; c* = {c_star}, C_max = {c_max}", flush=True)
    cal = [(i, 0, n) for (i, _, n) in serving.poisson_trace(16, 0.0, seed=11)]
    serving.run_trace(eng, h, cal, 64, 8, c_star, c_max, n_max=3)          # captures the CUDA graphs
    if args.c1_requests != 16:
        cal = [(i, 0, n) for (i, _, n) in serving.poisson_trace(args.c1_requests, 0.0, seed=11)]
    _, m = serving.run_trace(eng, h, cal, 64, 8, c_star, c_max, n_max=3, timeout_s=3600)
    c1 = m["images_per_s"]
    print(f"C1 = {c1:.3f} images/s", flush=True)
    res = dict(workload="SD-1.5-shaped 512² (latent 64×64), B_max 8, steps U{20..50}, g 7.5, DDIM, "
                        f"{args.requests} Poisson requests per load, λ = ρ·C₁ (C₁ from {args.c1_requests} requests "
                        f"at t = 0), precision {eng.precision}",
               c1_images_per_s=c1, c_star=c_star, c_max=c_max,
               table={f"{k}": v for k, v in sorted(tab.items())}, loads={})
    loads = [(str(rho), serving.poisson_trace(args.requests, rho * c1, seed=7)) for rho in args.rho]
    if args.burst:
        nb = args.requests // 2
        span = args.burst_span_s * 1e6 if args.burst_span_s > 0 else nb / (2.0 * c1) * 1e6
        loads.append(("burst", serving.burst_trace(args.requests, 0.5 * c1, frac=0.5, span_us=int(span), seed=7)))
    for rho, trace in loads:
        row = {}
        for name0 in args.arms:
          for vs in args.vae_sms:
            name = name0 if vs == 0 else f"{name0} | VAE on {vs} SMs"
            pol, abl, chunk = ARMS[name0]
            cs, cm = (c_star, c_max) if chunk else (1, 1)
            t1 = time.time()
            hv = part_tables[vs][0] if vs > 0 else h
            _, g = serving.run_trace(eng, hv, trace, 64, 8, cs, cm, n_max=3, policy=pol, ablation=abl,
                                     timeout_s=3600, vae_sms=vs)
            if vs > 0:
                g["partition_sms_unet_vae"] = part_tables[vs][1]
            sim = simulate(hv, trace, pol, abl, cs, cm) if not args.no_sim else \
                dict(images_per_s=0.0, mean_e2e_ms=0.0, p99_e2e_ms=0.0)
            row[name] = dict(gpu=g, virtual_clock=sim)
            print(f"rho {rho}: {name:26s} {g['images_per_s']:.3f} img/s, mean {g['mean_e2e_ms']:.0f} ms, "
                  f"P99 {g['p99_e2e_ms']:.0f} ms, skips {g['skipped_steps']} | sim {sim['images_per_s']:.3f} img/s, "
                  f"mean {sim['mean_e2e_ms']:.0f}, P99 {sim['p99_e2e_ms']:.0f} ({time.time() - t1:.0f} s)", flush=True)
        res["loads"][rho] = row
    B.lib().sd_table_free(h)
    eng.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()

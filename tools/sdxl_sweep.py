"""CFG#5-shaped serving on one B200: SDXL-base shapes at 1024² (latent 128×128), VAE
decode chunked into c ∈ {4, 8, 16} work-item ranges, Poisson traces at ρ·C₁, steps U{20..50}, g 7.5,
B_max 8 (the paper's P99-vs-chunks sweep, on 1 GPU instead of 8 — requests shard per GPU, so the
per-GPU numbers are the same). Per c the τ/δ table is profiled on the GPU (m ≤ 8,
n ≤ 2) and the controller is pinned to that c (c* = C_max = c).

  python tools/sdxl_sweep.py [--requests 24] [--rho 0.5 0.8 1.05] [--chunks 4 8 16]
"""
import argparse
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

LAT = 128


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=24)
    ap.add_argument("--rho", type=float, nargs="+", default=[0.5, 0.8, 1.05])
    ap.add_argument("--chunks", type=int, nargs="+", default=[4, 8, 16])
    ap.add_argument("--out", default="profiles/r01/sdxl_sweep.json")
    args = ap.parse_args()
    eng = Engine("sdxl", max_latent_hw=LAT, b_max=8, c_max=16)
    eng.set_uncond(torch.from_numpy(synth.uncond_embedding(0, 77, 2048)), torch.from_numpy(synth.uncond_pooled(0, 1280)))
    t0 = time.time()
    eng.warmup(LAT, LAT, 8, n_dec=2)
    prof = profiler.Profiler(eng, LAT, LAT, 8, reps=1)
    tab = prof.measure([1] + args.chunks, b_max=8, n_max=2)
    prof.close()
    h = profiler.to_table_handle(tab)
    solo_u, solo_v = tab[(1, 8, 0, 0)][0], tab[(1, 0, 1, 0)][0]
    print(f"profiled {len(tab)} entries in {time.time() - t0:.0f} s; solo UNet round (m=8) {solo_u / 1e3:.1f} ms, "
          f"solo decode {solo_v / 1e3:.1f} ms", flush=True)
    cal = [(i, 0, n) for (i, _, n) in serving.poisson_trace(12, 0.0, seed=11)]
    serving.run_trace(eng, h, cal, LAT, 8, 1, 1, n_max=2)
    _, m = serving.run_trace(eng, h, cal, LAT, 8, 1, 1, n_max=2)
    c1 = m["images_per_s"]
    print(f"C1 = {c1:.3f} images/s", flush=True)
    res = dict(workload=f"SDXL-base shapes 1024² (latent 128), {args.requests} Poisson requests per point, steps "
                        "U{20..50}, g 7.5, B_max 8, λ = ρ·C₁, controller pinned to c",
               c1_images_per_s=c1, solo_unet_round_us=solo_u, solo_decode_us=solo_v,
               inflation={f"c={c}": tab[(c, 8, 1, 0)][0] / (c * solo_u) for c in [1] + args.chunks},
               points=[])
    for rho in args.rho:
        trace = serving.poisson_trace(args.requests, rho * c1, seed=7)
        for c in args.chunks:
            _, g = serving.run_trace(eng, h, trace, LAT, 8, c, c, n_max=2, timeout_s=900)
            res["points"].append(dict(rho=rho, c=c, **g))
            print(f"rho {rho} c {c}: {g['images_per_s']:.3f} img/s, mean {g['mean_e2e_ms']:.0f} ms, "
                  f"P99 {g['p99_e2e_ms']:.0f} ms, skips {g['skipped_steps']}", flush=True)
    B.lib().sd_table_free(h)
    eng.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py — SynerDiff (arXiv 2605.08835) hot path on B200: images/s through libsynerdiff.so.

Workload (BASELINE.json configs[1] = SURVEY §8(d) CFG#2): SD-1.5-shaped UNet (random-init weights,
bf16), 512x512 images (latent 64x64), a batch of 8 requests per GPU denoised in lockstep for 50
DDIM steps with CFG on every step (16 UNet rows per sd_step_batch), then 8 whole-image VAE decodes.
One bench step = one pass of the whole hot path over one batch = 8 images per GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun (one process per GPU, NCCL); requests are sharded (weak scaling) and
the only collective on the serving path is the all-gather of per-rank queue loads.
`--impl reference` times the NumPy oracle (oracle/, the CPU reference of this tier) on a bounded
sample of the same workload and extrapolates images/s.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "images/sec (SD-1.5-shaped 512x512, 50 DDIM steps, CFG)"
UNIT = "images/s"
N_REQ = 8
N_STEPS = 50
G = 7.5
LAT = 64


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("bf16_tflops_sustained", 1417.2), d.get("bf16_tflops", 1681.1), d.get("hbm_gbs", 6446.9), \
            "measured (MEASURED_PEAKS.json)"
    return 1400.0, 1590.0, 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    def __init__(self, dev):
        self.dev = dev
        self.proc = None
        self.out = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.out.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.out:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------------
# reference arm: the oracle (NumPy, CPU) on a bounded sample
# ------------------------------------------------------------------------------------------------
def cpu_sample(steps=1, warmup=0, quiet=False):
    """Time the oracle: one SD-1.5 UNet row forward at 64x64 per step, plus one VAE decode at a 32x32
    latent scaled by 4 (pixel ratio; convs are 97 % of VAE work). images/s = 1/(100·t_row + 4·t_vae32)."""
    import numpy as np

    import synth
    from oracle import configs, unet, vae
    P = configs.unet_params(configs.SD15_UNET, 0, np.float32, bf16_weights=True)
    V = configs.vae_params(configs.SD_VAE, 0, np.float32, bf16_weights=True)
    x = synth.initial_noise(1, 0, LAT, LAT)[None]
    ctx = synth.text_embedding(1, 0, 77, 768)[None]
    z32 = synth.initial_noise(1, 0, 32, 32)[None]
    t0 = time.perf_counter()
    vae.decode(V, configs.SD_VAE, z32)
    t_vae = (time.perf_counter() - t0) * 4
    rows = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        unet.forward(P, configs.SD15_UNET, x, np.array([981]), ctx)
        if i >= warmup:
            rows.append(time.perf_counter() - t0)
    t_row = sum(rows) / len(rows)
    per_image = 2 * N_STEPS * t_row + t_vae
    return {"value": 1.0 / per_image, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
            "t_row_s": t_row, "t_vae_s": t_vae,
            "sample": f"{len(rows)} SD-1.5 UNet row forward(s) at latent 64x64 + 1 VAE decode at latent 32x32 "
                      f"(x4 pixel scaling); images/s = 1/(2*{N_STEPS}*t_row + t_vae), extrapolated"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t0 = time.perf_counter()
    cb = cpu_sample(steps=args.steps, warmup=min(args.warmup, 1))
    wall = time.perf_counter() - t0
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["t_row_s"] * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config(args.gpus), "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)


def config(n, precision="fp16"):
    return {"workload": "CFG#2: SD-1.5-shaped UNet (bf16-valued weights), 512x512 (latent 64x64), 8 requests/GPU "
                        "lockstep x 50 DDIM steps, CFG every step (16 UNet rows/step), then 8 whole VAE decodes "
                        "(on a low-priority stream, overlapping the next batch's UNet steps: PAPER.md:146-148; "
                        "--no-overlap serialises them)",
            "precision": f"{precision} tensor-core operands / activations, fp32 accumulation (DESIGN R19a)",
            "model": "sd15-shaped UNet (859.5M params) + SD VAE decoder, random init", "global_batch": N_REQ * n,
            "seq_len": LAT * LAT, "parallelism": f"dp{n} (request sharding, weak scaling)",
            "l2": "inputs larger than L2: 1.7 GB of UNet weights and >40 MB per activation stream through HBM"}


def serving_bench(eng, world, rank, args):
    """CFG#3-shaped serving on this GPU (and, for N > 1, every rank serves its shard id mod P with
    the per-rank loads all-gathered over NCCL for the controller — weak scaling):
      1. offline profiler: τ/δ table for c ∈ {1, 2}, m ≤ 8, n ≤ 3 on two streams (§III-C)
      2. C₁ = saturation throughput (16 requests arriving at t = 0)
      3. a Poisson trace at λ = ρ·C₁ per GPU, steps U{20..50}, g = 7.5 → images/s, mean / P99 E2E."""
    import torch
    import torch.distributed as dist

    from paper_2605_08835_b200 import binding as Bd
    from paper_2605_08835_b200 import profiler, serving
    t0 = time.perf_counter()
    eng.warmup(LAT, LAT, N_REQ, n_dec=3)  # every step-shape graph + pooled decode states, before any timing
    prof = profiler.Profiler(eng, LAT, LAT, N_REQ, reps=1)
    tab = prof.measure([1, 2], b_max=N_REQ, n_max=3)
    prof.close()
    h = profiler.to_table_handle(tab)
    c_max, c_star, _ = profiler.chunk_choice(tab, [1, 2], m=N_REQ, n=1)
    c_max = max(c_max, c_star)
    t_prof = time.perf_counter() - t0
    if world > 1:
        from paper_2605_08835_b200 import control_plane
        ctl = control_plane.LoadGather(eng, world, rank, group=args.ctl_group, device=rank)
    cal_trace = [(i, 0, n) for (i, _, n) in serving.poisson_trace(16, 0.0, seed=11)]
    # the first pass captures the CUDA graphs of the batch shapes the trace visits; the second is timed
    serving.run_trace(eng, h, cal_trace, LAT, N_REQ, c_star, c_max, n_max=3)
    _, cal = serving.run_trace(eng, h, cal_trace, LAT, N_REQ, c_star, c_max, n_max=3)
    c1 = cal["images_per_s"]
    full = serving.poisson_trace(args.serving_requests * world, args.rho * c1 * world, seed=7)
    mine_tr = [(i, a, n) for (i, a, n) in full if i % world == rank]
    if world > 1:
        ctl.start()
    _, m = serving.run_trace(eng, h, mine_tr, LAT, N_REQ, c_star, c_max, n_max=3)
    if world > 1:
        ctl.stop()  # leaves once every rank reported done (same number of collectives)
        m["allgather_us_mean"] = ctl.mean_us()
    Bd.lib().sd_table_free(h)
    out = {"workload": f"CFG#3-shaped: SD-1.5 512², Poisson λ = {args.rho}·C₁ per GPU, steps U{{20..50}}, g 7.5, "
                       f"controller on, c* = {c_star}, C_max = {c_max}, B_max = 8",
           "c1_images_per_s": c1, "rho": args.rho, "table_entries": len(tab), "profile_s": t_prof,
           "per_rank": m}
    if world > 1:
        vec = torch.tensor([m["images_per_s"], m["mean_e2e_ms"], m["p99_e2e_ms"]], dtype=torch.float64,
                           device=f"cuda:{rank}")
        g = [torch.zeros_like(vec) for _ in range(world)]
        dist.all_gather(g, vec)
        out["images_per_s"] = float(sum(x[0].item() for x in g))
        out["mean_e2e_ms"] = float(max(x[1].item() for x in g))
        out["p99_e2e_ms"] = float(max(x[2].item() for x in g))
    else:
        out.update(images_per_s=m["images_per_s"], mean_e2e_ms=m["mean_e2e_ms"], p99_e2e_ms=m["p99_e2e_ms"])
    return out


# ------------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--denoise-steps", type=int, default=N_STEPS)
    ap.add_argument("--precision", default="fp16", choices=["bf16", "fp16"],
                    help="16-bit operand / storage type of the UNet and VAE kernels (fp32 accumulation either way; "
                         "the weights are the bf16 values of R20 in both). fp16 (default): the paper's FP16 (P:315), "
                         "8x lower error than bf16 at the same tensor-core rate")
    ap.add_argument("--no-alt-precision", action="store_true",
                    help="skip the second timed leg in the other 16-bit precision")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-serving", action="store_true")
    ap.add_argument("--no-overlap", action="store_true",
                    help="decode each batch on the UNet stream after its last step instead of on the "
                         "low-priority VAE stream overlapping the next batch's UNet steps")
    ap.add_argument("--serving-requests", type=int, default=200)
    ap.add_argument("--rho", type=float, default=0.8)
    ap.add_argument("--profile-range", action="store_true",
                    help="bracket the timed region with cudaProfilerStart/Stop (ncu --profile-from-start off)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2605_08835_b200.engine import Engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    args.ctl_group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        # C1 runs on its own communicator (and, in control_plane, its own stream and thread), so the
        # lockstep data plane below never waits on a peer
        args.ctl_group = dist.new_group(backend="nccl")
    dev = torch.device(f"cuda:{local}")
    nsteps = args.denoise_steps

    eng = Engine("sd15", max_latent_hw=LAT, b_max=N_REQ, device=local, precision=args.precision)
    eng.set_uncond(torch.from_numpy(synth.uncond_embedding(0, 77, 768)))
    # UNet steps on a high-priority stream; each batch's decodes on a low-priority one, overlapping the
    # next batch's UNet steps (the paper's UNet ∥ VAE co-execution, at batch granularity)
    st = torch.cuda.Stream(device=dev, priority=-1)
    vst = torch.cuda.Stream(device=dev, priority=0)
    ids = [rank * N_REQ + i for i in range(N_REQ)]
    # host inputs (pinned): text embeddings and initial noise per request (R20)
    emb_h = torch.from_numpy(np.stack([synth.text_embedding(1, i, 77, 768) for i in ids])).pin_memory()
    z_h = torch.from_numpy(np.stack([synth.initial_noise(1, i, LAT, LAT) for i in ids])).pin_memory()
    img_h = torch.empty(N_REQ, 3, 8 * LAT, 8 * LAT, dtype=torch.float32).pin_memory()
    # device-resident inputs for the kernel-throughput number
    emb_d = emb_h.to(dev)
    z_d = z_h.to(dev)
    slots = [eng.register(emb_d[i]) for i in range(N_REQ)]
    lats = [torch.empty_like(z_d), torch.empty_like(z_d)]  # batch k uses lats[k % 2]
    imgs = torch.empty(N_REQ, 3, 8 * LAT, 8 * LAT, device=dev)
    pipe = {"k": 0, "dec": [None, None], "last": None}

    def denoise_and_decode(slot_ids, overlap=not args.no_overlap):
        """One bench step (8 requests: 50 steps + 8 decodes). With overlap, the decodes go to the
        low-priority stream after this batch's last UNet step, and the next batch's UNet steps start at
        once on `st` (the latents buffer is double-buffered; a batch waits for the decodes of the batch two
        back, which read the same buffer). `drain()` makes `st` wait for the outstanding decodes."""
        b = pipe["k"] % 2
        pipe["k"] += 1
        lat = lats[b]
        with torch.cuda.stream(st):
            if pipe["dec"][b] is not None:
                st.wait_event(pipe["dec"][b])
            lat.copy_(z_d)                       # x_T = init_sigma (=1, DDIM) · z
            views = [lat[i] for i in range(N_REQ)]
            for s in range(nsteps):
                eng.step(views, [s] * N_REQ, [nsteps] * N_REQ, [1] * N_REQ, [G] * N_REQ, slot_ids, stream=st)
            if not overlap:
                for i in range(N_REQ):
                    eng.decode(lat[i], 1, image=imgs[i], stream=st)
                pipe["dec"][b] = None
                return
            done = torch.cuda.Event()
            done.record(st)
        with torch.cuda.stream(vst):
            vst.wait_event(done)
            for i in range(N_REQ):
                eng.decode(lat[i], 1, image=imgs[i], stream=vst)
            ev = torch.cuda.Event()
            ev.record(vst)
        pipe["dec"][b] = ev
        pipe["last"] = ev

    def drain():
        if pipe["last"] is not None:
            st.wait_event(pipe["last"])

    for _ in range(args.warmup):
        denoise_and_decode(slots)
    torch.cuda.synchronize()

    # ---- device-resident timed region ----
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = eng.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        if args.profile_range:
            torch.cuda.cudart().cudaProfilerStart()
        ev0.record(st)
        for _ in range(args.steps):
            denoise_and_decode(slots)
        drain()  # the last batch's decodes are inside the timed region
        ev1.record(st)
        torch.cuda.synchronize()
        if args.profile_range:
            torch.cuda.cudart().cudaProfilerStop()
    if world > 1:
        dist.barrier()
    n_launch = eng.launch_count() - n0
    ms = ev0.elapsed_time(ev1)
    # per-kernel-class device times: the same K steps again with CUDA events around every launch on
    # the launching stream (eager launches; kernel durations are those of the graph replays above)
    torch.cuda.synchronize()
    eng.profile(True)
    with torch.cuda.stream(st):
        for _ in range(args.steps):
            denoise_and_decode(slots, overlap=False)  # per-class times without co-running kernels
    torch.cuda.synchronize()
    prof = {c: eng.profile_read(c) for c in (0, 1, 2, 3, 4, 7)}
    eng.profile(False)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = N_REQ * world * args.steps / (ms_max / 1e3)

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        h2d = emb_h.numel() * 4 + z_h.numel() * 4
        d2h = img_h.numel() * 4
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        prev = None
        for _ in range(args.steps):
            with torch.cuda.stream(st):
                emb_d.copy_(emb_h, non_blocking=True)
                z_d.copy_(z_h, non_blocking=True)
            sl = [eng.register(emb_d[i], stream=st) for i in range(N_REQ)]
            denoise_and_decode(sl)
            # the images of this batch leave once its decodes are done (on the decode stream when
            # overlapped); the host waits for the previous batch only, so batches pipeline
            dstream = st if args.no_overlap else vst
            with torch.cuda.stream(dstream):
                img_h.copy_(imgs, non_blocking=True)
                out_ev = torch.cuda.Event()
                out_ev.record(dstream)
            st.synchronize()  # this batch's UNet steps (its text K/V slots are then free to reuse)
            for s_ in sl:
                eng.release(s_)
            if prev is not None:
                prev.synchronize()
            prev = out_ev
        drain()
        if prev is not None:
            st.wait_event(prev)
        e1.record(st)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": N_REQ * world * args.steps / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "note": "per step: H2D of 8 prompt embeddings + 8 noise latents (pinned), text K/V admission, "
                       "50 steps, 8 decodes, D2H of 8 images"}

    # ---- continuous-batching serving (CFG#3 shape): offline profile → trace → mean / P99 E2E ----
    serving_out = None
    if not args.no_serving:
        try:
            serving_out = serving_bench(eng, world, rank, args)
        except Exception as ex:  # the serving leg must never sink the bench line
            serving_out = {"error": repr(ex)}

    # ---- the same device-resident step in the other 16-bit precision (same kernels; BASELINE's config
    # names bf16, the product default is fp16 — both are reported, the headline is --precision) ----
    alt = None
    if not args.no_alt_precision:
        for s_ in slots:
            eng.release(s_)
        eng.close()
        torch.cuda.synchronize()
        other = "bf16" if args.precision == "fp16" else "fp16"
        eng = Engine("sd15", max_latent_hw=LAT, b_max=N_REQ, device=local, precision=other)
        eng.set_uncond(torch.from_numpy(synth.uncond_embedding(0, 77, 768)))
        slots = [eng.register(emb_d[i]) for i in range(N_REQ)]
        for _ in range(args.warmup):
            denoise_and_decode(slots)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        for _ in range(args.steps):
            denoise_and_decode(slots)
        drain()
        a1.record(st)
        torch.cuda.synchronize()
        ta = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ta, op=dist.ReduceOp.MAX)
        alt = {"dtype": other, "value": N_REQ * world * args.steps / (float(ta.item()) / 1e3), "unit": UNIT,
               "ms_per_step": float(ta.item()) / args.steps,
               "note": "same workload, kernels and timing rules; only the 16-bit operand / storage type differs"}

    if rank == 0:
        sus, burst, hbm, src = peaks()
        conv_ms, conv_n, conv_flops = prof[0]
        achieved = conv_flops / (conv_ms / 1e3) / 1e12 if conv_ms > 0 else 0.0
        kern = {}
        for c, name in enumerate(["conv3x3_implicit_gemm", "dense_gemm", "attention", "groupnorm", "layernorm"]):
            m_, n_, w_ = prof[c]
            rate = w_ / (m_ / 1e3) if m_ > 0 else 0.0
            kern[name] = {"ms_per_step": m_ / args.steps, "launches": n_,
                          ("tflops" if c < 3 else "gbs"): rate / (1e12 if c < 3 else 1e9)}
        m7, n7, w7 = prof[7]
        kern["conv1x1_gemm"] = {"ms_per_step": m7 / args.steps, "launches": n7,
                                "tflops": w7 / (m7 / 1e3) / 1e12 if m7 > 0 else 0.0}
        # SURVEY §8(d) UNet conv fraction: conv3x3/up/down AND the 1×1 shortcut / proj_in / proj_out convs
        conv_all = (conv_flops + w7) / ((conv_ms + m7) / 1e3) / 1e12 if conv_ms + m7 > 0 else 0.0
        traffic = None
        tp = os.path.join(ROOT, "profiles", "conv_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.precision, "data": "synthetic (seeded; random-init weights)",
            "config": config(world, args.precision),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": sus, "unit": "TFLOP/s",
                         "frac": achieved / sus, "traffic": traffic,
                         "kernel": "conv3x3 implicit GEMM (tcgen05/TMEM/TMA), all UNet conv3x3 launches",
                         "peak_source": f"{src}, sustained bf16 (kernel timed inside a long step)",
                         "launches": conv_n, "flops_per_launch": conv_flops / max(conv_n, 1),
                         "unet_conv_all": {"achieved": conv_all, "frac": conv_all / sus,
                                           "gflop_per_unet_step": (conv_flops + w7) / args.steps / args.denoise_steps / 1e9,
                                           "note": "SURVEY 8(d) definition: conv3x3 + 1x1 shortcut / proj_in / "
                                                   "proj_out, all UNet launches"}},
            "kernels": kern,
            "e2e": e2e,
            "gpu_launches": n_launch,
            "clocks": clk.summary(),
            "latency_ms": {
                "mean_e2e": (serving_out or {}).get("mean_e2e_ms"), "p99_e2e": (serving_out or {}).get("p99_e2e_ms"),
                "lockstep_ms_per_step": ms_max / args.steps,
                "note": "E2E (V_i - A_i, R18) mean / P99 of the serving leg (CFG#3-shaped Poisson trace at rho "
                        "C1, see serving); the lockstep step completes all 8 images together"},
            "serving": serving_out,
            "precision_alt": alt,
            "precision_note": ("fp16 = fp16 operands / activations with the bf16-valued R20 weights held exactly; "
                               "fp32 accumulation, statistics, latents and eps in both"),
        }
        if not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_sample(steps=1)
            except Exception as ex:  # the baseline must never sink the bench line
                line["cpu_baseline"] = {"error": repr(ex)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    eng.close()


if __name__ == "__main__":
    main()

"""Host-timed phases of bench.py's end-to-end leg (diagnostic): admission (sd_ctx_register × 8),
50 sd_step_batch calls, 8 whole decodes, D2H — each phase synchronised, wall-clock per phase.

  python tools/e2e_probe.py [--iters 3]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_08835_b200.engine import Engine  # noqa: E402

N, LAT, STEPS = 8, 64, 50


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    eng = Engine("sd15", max_latent_hw=LAT, b_max=N)
    eng.set_uncond(torch.from_numpy(synth.uncond_embedding(0, 77, 768)))
    st = torch.cuda.Stream(device=dev)
    emb_h = torch.from_numpy(np.stack([synth.text_embedding(1, i, 77, 768) for i in range(N)])).pin_memory()
    z_h = torch.from_numpy(np.stack([synth.initial_noise(1, i, LAT, LAT) for i in range(N)])).pin_memory()
    img_h = torch.empty(N, 3, 8 * LAT, 8 * LAT).pin_memory()
    emb_d, z_d = emb_h.to(dev), z_h.to(dev)
    lat = torch.empty_like(z_d)
    imgs = torch.empty(N, 3, 8 * LAT, 8 * LAT, device=dev)
    for it in range(args.iters):
        t = [time.perf_counter()]
        with torch.cuda.stream(st):
            emb_d.copy_(emb_h, non_blocking=True)
            z_d.copy_(z_h, non_blocking=True)
        sl = [eng.register(emb_d[i], stream=st) for i in range(N)]
        st.synchronize()
        t.append(time.perf_counter())
        with torch.cuda.stream(st):
            lat.copy_(z_d)
        views = [lat[i] for i in range(N)]
        for s in range(STEPS):
            eng.step(views, [s] * N, [STEPS] * N, [1] * N, [7.5] * N, sl, stream=st)
        t.append(time.perf_counter())
        st.synchronize()
        t.append(time.perf_counter())
        for i in range(N):
            eng.decode(lat[i], 1, image=imgs[i], stream=st)
        t.append(time.perf_counter())
        st.synchronize()
        t.append(time.perf_counter())
        with torch.cuda.stream(st):
            img_h.copy_(imgs, non_blocking=True)
        st.synchronize()
        t.append(time.perf_counter())
        for s_ in sl:
            eng.release(s_)
        d = np.diff(t) * 1e3
        print(f"iter {it}: register {d[0]:.1f} ms | steps enqueue {d[1]:.1f} + drain {d[2]:.1f} | decode enqueue "
              f"{d[3]:.1f} + drain {d[4]:.1f} | D2H {d[5]:.1f} | total {sum(d):.1f} ms", flush=True)


if __name__ == "__main__":
    main()

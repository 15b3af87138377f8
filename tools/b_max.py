"""B_max from the profiler's saturation rule on the B200 ("we identify the saturation batch
size B_max based on the sub-linear scaling of throughput"; SPEC find_b_max):
τ^1(m, 0, 0) for m = 1 … M (one UNet step of m requests, CFG rows 2m, CUDA graphs) measured by the
offline profiler on the high-priority stream, then sd_find_b_max with ε = 0.05.

  python tools/b_max.py [--model sd15] [--latent 64] [--m-max 16] [--out profiles/r02/b_max_sd15_512.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_08835_b200 import profiler  # noqa: E402
from paper_2605_08835_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="sd15")
    ap.add_argument("--latent", type=int, default=64)
    ap.add_argument("--m-max", type=int, default=16)
    ap.add_argument("--precision", default="fp16")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    eng = Engine(a.model, max_latent_hw=a.latent, b_max=a.m_max, c_max=2, precision=a.precision)
    L, D = eng.ctx_len, eng.ctx_dim
    eng.set_uncond(torch.from_numpy(synth.uncond_embedding(0, L, D)),
                   torch.from_numpy(synth.uncond_pooled(0, eng.pooled_dim)) if eng.pooled_dim else None)
    t0 = time.time()
    # the first measurement of each m captures its CUDA graph; the median of 5 excludes it
    prof = profiler.Profiler(eng, a.latent, a.latent, a.m_max, reps=3)
    tab = profiler.solo_unet_table(prof, a.m_max, reps=5)
    prof.close()
    res = {"model": a.model, "latent": a.latent, "precision": a.precision, "eps": 0.05,
           "tau_us": {m: tab[(1, m, 0, 0)][0] for m in range(1, a.m_max + 1)},
           "images_per_s_per_step": {m: m / (tab[(1, m, 0, 0)][0] / 1e6) for m in range(1, a.m_max + 1)}}
    res["b_max"] = profiler.find_b_max(tab, a.m_max, (1, 20))
    res["profile_s"] = time.time() - t0
    line = json.dumps(res)
    print(line, flush=True)
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        open(a.out, "w").write(line + "\n")
    eng.close()


if __name__ == "__main__":
    main()

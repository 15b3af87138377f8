"""One denoising step of the bench workload (8 requests × CFG = 16 UNet rows, SD-1.5 shape, 64×64
latents) inside a cudaProfilerStart/Stop range, for `ncu --profile-from-start off --set full
-k regex:<kernel>` captures of the kernels as bench.py launches them (same shapes, same graphs).

  ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:gemm_kernel -o gpurun_out/conv python tools/ncu_step.py [--decode]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2605_08835_b200.engine import Engine  # noqa: E402

N_REQ, LAT, G, STEPS = 8, 64, 7.5, 50


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--decode", action="store_true", help="profile one VAE decode instead of a UNet step")
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    eng = Engine("sd15", max_latent_hw=LAT, b_max=N_REQ, device=0)
    eng.set_uncond(torch.from_numpy(synth.uncond_embedding(0, 77, 768)))
    st = torch.cuda.Stream(device=dev)
    emb = torch.from_numpy(np.stack([synth.text_embedding(1, i, 77, 768) for i in range(N_REQ)])).to(dev)
    lat = torch.from_numpy(np.stack([synth.initial_noise(1, i, LAT, LAT) for i in range(N_REQ)])).to(dev)
    slots = [eng.register(emb[i]) for i in range(N_REQ)]
    img = torch.empty(3, 8 * LAT, 8 * LAT, device=dev)
    views = [lat[i] for i in range(N_REQ)]

    def one():
        with torch.cuda.stream(st):
            if args.decode:
                eng.decode(lat[0], 1, image=img, stream=st)
            else:
                eng.step(views, [0] * N_REQ, [STEPS] * N_REQ, [1] * N_REQ, [G] * N_REQ, slots, stream=st)

    for _ in range(args.warmup):
        one()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    one()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("ok")


if __name__ == "__main__":
    main()

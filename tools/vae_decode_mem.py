"""SD VAE decode at 512² and 1024² on B200: time per whole / 4-chunk decode (CUDA events) and the device
memory a decode state takes (cudaMemGetInfo before / after the first decode of that size — the
DecodeState arena: activations, GN workspace and the query-chunked mid-attention scratch, whose fp32
scores are capped at 64 MB instead of a P×P matrix: 1 GiB at 1024²).

  python tools/vae_decode_mem.py [--out profiles/r02/vae_decode_mem.json]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_08835_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r02/vae_decode_mem.json")
    ap.add_argument("--precision", default="fp16")
    args = ap.parse_args()
    eng = Engine("sd15", max_latent_hw=128, b_max=1, c_max=16, precision=args.precision)
    rows = []
    for hw in (64, 128):
        z = torch.from_numpy(synth.initial_noise(3, hw, hw, hw)).cuda()
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
        eng.decode(z, 1)
        torch.cuda.synchronize()
        free1 = torch.cuda.mem_get_info()[0]
        for c in (1, 4):
            eng.decode(z, c)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                eng.decode(z, c)
            e1.record()
            torch.cuda.synchronize()
            rows.append(dict(latent=hw, image=8 * hw, chunks=c, ms=e0.elapsed_time(e1) / 5,
                             decode_state_mib=(free0 - free1) / 2 ** 20))
            print(json.dumps(rows[-1]), flush=True)
    eng.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(dict(what=__doc__.strip().splitlines()[0], precision=args.precision, rows=rows), open(args.out, "w"),
              indent=1)


if __name__ == "__main__":
    main()

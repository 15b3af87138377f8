"""V2 independent-tile VAE decode (R7 V2) vs the exact decode on B200: the
error-vs-halo curve (rel-L2 of the stitched image against the whole decode of the same latent) and
the decode time, beside the whole decode and the exact V1 chunked decode (c = 4), for the SD VAE at
latent 64×64 (512²) and 128×128 (1024²).

  python tools/vae_tiles.py [--out profiles/r01/vae_v2_tiles.json]
"""
import argparse
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_08835_b200.engine import Engine  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r01/vae_v2_tiles.json")
    args = ap.parse_args()
    res = {"what": "rel-L2 of the V2 stitched image vs the whole decode of the same latent (bf16 GPU path); "
                   "ms per decode (CUDA events, 3 reps after a warm-up)", "rows": []}
    eng = Engine("sd15", max_latent_hw=128, b_max=1, c_max=16)
    for hw in (64, 128):
        z = torch.from_numpy(synth.initial_noise(3, hw, hw, hw)).cuda()
        whole, t_whole = timed(lambda: eng.decode(z, 1))
        chunked, t_v1 = timed(lambda: eng.decode(z, 4))
        assert torch.equal(chunked, whole)
        res["rows"].append(dict(latent=hw, mode="whole", ms=t_whole))
        res["rows"].append(dict(latent=hw, mode="V1 chunked c=4 (exact)", ms=t_v1, rel_l2=0.0))
        nrm = whole.double().norm().item()
        for tile in (16, 32):
            for halo in (0, 8, 16, 24):
                img, t = timed(lambda: eng.decode_tiled(z, tile, halo))
                err = (img.double() - whole.double()).norm().item() / nrm
                res["rows"].append(dict(latent=hw, mode=f"V2 tile {tile} halo {halo}", tile=tile, halo=halo,
                                        ms=t, rel_l2=err))
                print(f"latent {hw}: tile {tile} halo {halo}: rel-L2 {err:.3e}, {t:.2f} ms "
                      f"(whole {t_whole:.2f} ms, V1 c=4 {t_v1:.2f} ms)", flush=True)
    eng.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

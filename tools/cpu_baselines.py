"""CPU-oracle baselines of SURVEY §8(d) / BASELINE.md §4, timed on the GPU box's own host cores
(the oracle as it stands, NumPy fp32, BLAS threads = all cores). Items:

  CFG#1 end to end   tiny UNet, 2 requests x 4 DDIM steps with CFG (g 7.5), 2-chunk VAE decode each
  SD-1.5 512^2       one UNet row forward (latent 64^2) and one whole VAE decode (512^2)
  SD-1.5 768^2       one UNet row forward (latent 96^2) and one whole VAE decode (768^2)
  SDXL 1024^2        one UNet row forward (latent 128^2) and one whole VAE decode (1024^2)

and the per-image extrapolation (n = 50 steps, CFG every step: 2n row forwards + 1 decode), labelled as
such. Writes one JSON object (stdout, and --out). Test infrastructure: imports oracle/ (allowed here:
this is the cpu_baseline leg of the measurement, not the product path).
Usage: python tools/cpu_baselines.py [--out profiles/r02/cpu_baselines.json] [--skip-sdxl]"""
import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import configs, pipeline, sampling, unet, vae  # noqa: E402


def timed(fn):
    t0 = time.perf_counter()
    out = fn()
    return time.perf_counter() - t0, out


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 0) for i in threadpool_info()), default=None)
    except Exception:
        return None


def cfg1_end_to_end():
    P = configs.unet_params(configs.TINY_UNET, 0, np.float32, bf16_weights=True)
    V = configs.vae_params(configs.TINY_VAE, 0, np.float32, bf16_weights=True)
    cu = synth.bf16_round(synth.uncond_embedding(0, 8, 32))

    def run():
        for i in range(2):
            x = pipeline.denoise(P, configs.TINY_UNET, synth.initial_noise(1, i, 8, 8),
                                 synth.bf16_round(synth.text_embedding(1, i, 8, 32)), cu, 4, 7.5, "ddim")
            vae.decode_chunked(V, configs.TINY_VAE, x[None], n_chunks=2)
    return timed(run)[0]


def row_and_decode(ucfg, vcfg, lat, ctx_len, ctx_dim, pooled_dim):
    P = configs.unet_params(ucfg, 0, np.float32, bf16_weights=True)
    x = synth.initial_noise(1, 0, lat, lat)[None]
    ctx = synth.text_embedding(1, 0, ctx_len, ctx_dim)[None]
    kw = {}
    if pooled_dim:
        kw["pooled"] = synth.pooled_embedding(1, 0, pooled_dim)[None]
    t = int(sampling.timesteps(50)[0])
    t_row, _ = timed(lambda: unet.forward(P, ucfg, x, np.array([t]), ctx, **kw))
    del P
    V = configs.vae_params(vcfg, 0, np.float32, bf16_weights=True)
    z = synth.initial_noise(3, 0, lat, lat)[None]
    t_vae, _ = timed(lambda: vae.decode(V, vcfg, z))
    return t_row, t_vae


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--skip-sdxl", action="store_true")
    args = ap.parse_args()
    res = {"kind": "oracle (NumPy fp32, as it stands)", "cores": os.cpu_count(), "blas_threads": blas_threads(),
           "cpu_model": cpu_model(), "items": {}}
    t = cfg1_end_to_end()
    res["items"]["cfg1_end_to_end_s"] = t
    print(f"CFG#1 end to end: {t:.2f} s", flush=True)
    work = [("sd15_512", configs.SD15_UNET, configs.SD_VAE, 64, 77, 768, 0, 803.2, 2514.5),
            ("sd15_768", configs.SD15_UNET, configs.SD_VAE, 96, 77, 768, 0, 2148.1, 5754.3)]
    if not args.skip_sdxl:
        work.append(("sdxl_1024", configs.SDXL_UNET, configs.SD_VAE, 128, 77, 2048, 1280, 6761.2, 10470.4))
    for name, uc, vc, lat, L, D, PD, gf_row, gf_vae in work:
        t_row, t_vae = row_and_decode(uc, vc, lat, L, D, PD)
        per_image = 2 * 50 * t_row + t_vae
        res["items"][name] = {"row_forward_s": t_row, "vae_decode_s": t_vae,
                              "row_gflops_per_s": gf_row / t_row, "vae_gflops_per_s": gf_vae / t_vae,
                              "images_per_s_extrapolated": 1.0 / per_image,
                              "extrapolation": "1 / (2*50*t_row + t_vae): 50 DDIM steps with CFG every step"}
        print(f"{name}: row {t_row:.1f} s, decode {t_vae:.1f} s -> {1.0 / per_image:.3e} images/s (extrapolated)",
              flush=True)
    line = json.dumps(res)
    print(line)
    if args.out:
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()

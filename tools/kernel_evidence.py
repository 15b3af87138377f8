"""Per-kernel-class ncu evidence for one 16-row SD-1.5 UNet step and one 512² VAE decode (the bench
workload), as the north star asks: tensor-pipe utilisation for the convs, GEMMs and attention;
achieved DRAM GB/s for norms, combine and the VAE against the chip's measured peak.

  ncu --metrics <METRICS> --cache-control none --clock-control none --profile-from-start off --csv \\
      --log-file gpurun_out/ev_step.csv python tools/ncu_step.py
  ncu ... --log-file gpurun_out/ev_vae.csv python tools/ncu_step.py --decode
  python tools/kernel_evidence.py gpurun_out/ev_step.csv gpurun_out/ev_vae.csv > profiles/r01/kernel_evidence.json

Warm caches (--cache-control none): the kernels run as in the step, producer outputs partly L2-resident.
"""
import collections
import csv
import json
import re
import os
import sys

METRICS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,"
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,launch__grid_size")



def gemm_mode(name):
    """MODE template argument (0 dense, 1 conv3) of a gemm_kernel<BN, CG, MODE[, F16]> name, else None."""
    m = re.search(r"gemm_kernel<\s*(\d+)\s*,\s*(\d+)\s*,\s*(\d+)", name)
    return int(m.group(3)) if m else None

def classify(name):
    n = name.split("(")[0]
    if "gemm_kernel" in n:
        return "conv3x3 implicit GEMM (tcgen05)" if gemm_mode(name) == 1 else "dense GEMM (tcgen05)"
    if "xattn_tc_kernel" in n:
        return "cross-attention (tcgen05, K/V resident)"
    if "attn_tc" in n:
        return "self-attention (tcgen05 flash)"
    if "xattn" in n:
        return "cross-attention (short-context mma.sync)"
    if "attn_kernel" in n:
        return "self-attention (mma.sync flash)"
    if "gn_" in n:
        return "GroupNorm (stats/finalize/apply)"
    if "layer_norm" in n:
        return "LayerNorm"
    if "combine" in n or "gather_rows" in n:
        return "CFG gather + combine/sampler (K11/K12)"
    if "softmax_rows" in n:
        return "VAE attention softmax"
    return "other elementwise (concat, upsample, split-K reduce, layout)"


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.defaultdict(dict)
    scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1.0, "": 1.0}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        except ValueError:
            continue
        per[int(r[ii])][r[mi]] = v
        per[int(r[ii])]["name"] = r[ki]
    return [per[i] for i in sorted(per)]


def summarize(launches, hbm_gbs):
    agg = collections.defaultdict(lambda: dict(launches=0, us=0.0, bytes=0.0, tensor_w=0.0, xu_w=0.0))
    for d in launches:
        c = classify(d["name"])
        a = agg[c]
        t = d.get("gpu__time_duration.sum", 0.0)
        a["launches"] += 1
        a["us"] += t
        a["bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        a["tensor_w"] += t * d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
        a["xu_w"] += t * d.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 0.0)
    tot = sum(a["us"] for a in agg.values())
    out = []
    for c, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
        gbs = a["bytes"] / (a["us"] * 1e-6) / 1e9 if a["us"] else 0.0
        out.append(dict(kernel_class=c, launches=a["launches"], us=round(a["us"], 1), share=round(a["us"] / tot, 4),
                        tensor_pipe_pct=round(a["tensor_w"] / a["us"], 1) if a["us"] else 0.0,
                        mufu_xu_pct=round(a["xu_w"] / a["us"], 1) if a["us"] else 0.0,
                        dram_gbs=round(gbs, 1), dram_frac_of_peak=round(gbs / hbm_gbs, 3)))
    return dict(total_us=round(tot, 1), classes=out)


def main():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    hbm = 6446.9
    p = os.path.join(root, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        hbm = json.load(open(p)).get("hbm_gbs", hbm)
    res = {"how": "ncu --metrics " + METRICS + " --cache-control none --clock-control none over tools/ncu_step.py "
                  "(one 16-row SD-1.5 512² UNet step; one 512² VAE decode); tensor/MUFU % time-weighted per class; "
                  "DRAM GB/s = (dram read + write bytes) / kernel time",
           "hbm_peak_gbs": hbm}
    for label, path in zip(("unet_step", "vae_decode"), sys.argv[1:3]):
        res[label] = summarize(load(path), hbm)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

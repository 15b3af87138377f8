"""DRAM traffic per conv3x3 op of one 16-row SD-1.5 UNet step, from an `ncu --set full` capture of the
GEMM kernels (the bench roofline's `traffic` field reads profiles/conv_traffic.json).

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\\
        sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --cache-control all \\
      --clock-control none --profile-from-start off -k regex:"gemm_kernel|splitk_reduce" --csv --page raw \\
      --log-file gpurun_out/conv_cold.csv python tools/ncu_step.py
  python tools/conv_traffic.py gpurun_out/conv_cold.csv > profiles/conv_traffic.json
(a .ncu-rep from `ncu --set full` works too; --cache-control all = the same cold caches as --set full)

A conv op is one gemm_kernel<*,*,1> launch (+ the splitk_reduce_kernel that follows a split-K conv).
Cold caches (ncu's default cache control), serialised launches.
"""
import csv
import io
import json
import re
import subprocess
import sys



def gemm_mode(name):
    """MODE template argument (0 dense, 1 conv3) of a gemm_kernel<BN, CG, MODE[, F16]> name, else None."""
    m = re.search(r"gemm_kernel<\s*(\d+)\s*,\s*(\d+)\s*,\s*(\d+)", name)
    return int(m.group(3)) if m else None

def main():
    if sys.argv[1].endswith(".ncu-rep"):
        out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    else:
        out = open(sys.argv[1]).read()
    rows = list(csv.reader(io.StringIO(out)))
    rows = rows[next(i for i, r in enumerate(rows) if "Kernel Name" in r):]
    h, units = rows[0], rows[1]

    def val(r, m):
        i = h.index(m)
        v = float(r[i].replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
                    "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3, "%": 1.0}.get(units[i], 1.0)

    ops, cur = [], None
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        by = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        us = val(r, "gpu__time_duration.sum")
        tens = val(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
        base = name.split("(")[0]
        if gemm_mode(base) == 1:
            cur = dict(bytes=by, us=us, tensor_w=tens * us, launches=1)
            ops.append(cur)
        elif gemm_mode(base) == 0:
            cur = None  # a reduce after a dense GEMM (dense split-K) belongs to that GEMM, not to a conv
        elif "splitk_reduce" in base and cur is not None:
            cur["bytes"] += by
            cur["us"] += us
            cur["launches"] += 1
    n = len(ops)
    res = {
        "source": "ncu --cache-control all --clock-control none (cold cache, serialised) of the conv3x3 ops of one 16-row "
                  "SD-1.5 UNet step (tools/ncu_step.py); a conv op = gemm_kernel<*,*,1> (+ splitk_reduce_kernel "
                  "for split-K 8x8 convs); tools/conv_traffic.py",
        "conv_ops": n,
        "launches": sum(o["launches"] for o in ops),
        "dram_bytes_per_launch": sum(o["bytes"] for o in ops) / max(n, 1),
        "ncu_ms_per_unet_step": sum(o["us"] for o in ops) / 1e3,
        "mean_tensor_pipe_active_pct": sum(o["tensor_w"] for o in ops) / max(sum(o["us"] for o in ops), 1e-9),
        "round": "r02",
    }
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

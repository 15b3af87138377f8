"""Kernel micro-benchmarks on the B200 (CUDA events, warm L2 unless --flush): the SD-1.5 512² conv3x3
shapes at 16 rows and the big dense GEMMs, through the test-only C-ABI exports. Prints TFLOP/s per
shape and the fraction of the measured sustained bf16 peak.

  python tools/kbench.py [--reps 20] [--only conv|gemm]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_08835_b200 import binding as B  # noqa: E402

CONV = [  # (rows, H, W, Cin, Cout, count per UNet step)
    (16, 64, 64, 320, 320, 7), (16, 32, 32, 640, 640, 6), (16, 16, 16, 1280, 1280, 6), (16, 8, 8, 1280, 1280, 11),
    (16, 64, 64, 640, 320, 2), (16, 32, 32, 1280, 640, 1), (16, 16, 16, 2560, 1280, 2), (16, 8, 8, 2560, 1280, 3),
    (16, 64, 64, 640, 640, 1), (16, 32, 32, 1280, 1280, 1), (16, 64, 64, 960, 320, 2), (16, 32, 32, 1920, 640, 1),
]
VAE = [  # SD VAE decoder convs at 512² (one image, B = 1): (rows, H, W, Cin, Cout, count per decode)
    (1, 64, 64, 512, 512, 8), (1, 128, 128, 512, 512, 7), (1, 256, 256, 512, 256, 1), (1, 256, 256, 256, 256, 6),
    (1, 512, 512, 256, 128, 1), (1, 512, 512, 128, 128, 5),
]
GEMM = [  # (M, N, K, act)
    (65536, 2560, 320, 2), (65536, 320, 1280, 0), (65536, 960, 320, 0), (65536, 320, 320, 0),
    (16384, 5120, 640, 2), (16384, 640, 2560, 0), (4096, 10240, 1280, 2), (4096, 1280, 5120, 0),
    # 32×32 / 16×16 / 8×8 transformer projections (16 rows)
    (16384, 640, 640, 0), (16384, 1280, 640, 0), (4096, 1280, 1280, 0), (4096, 2560, 1280, 0),
    (1024, 1280, 1280, 0), (1024, 10240, 1280, 2),
]


def cur():
    return torch.cuda.current_stream().cuda_stream


def timeit(fn, reps):
    """Device time per call: `reps` calls captured in one CUDA graph (no host launch overhead)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="")
    ap.add_argument("--pick", type=int, default=-1, help="run only entry i of the selected list")
    args = ap.parse_args()
    peak = 1417.2
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peak = json.load(open(p)).get("bf16_tflops_sustained", peak)
    out = []
    tot_t = tot_f = 0.0
    for which, LIST in (("conv", CONV), ("vae", VAE)):
        if args.only not in ("", which):
            continue
        tot_t = tot_f = 0.0
        for i_, (R, H, W, ci, co, cnt) in enumerate(LIST):
            if args.pick >= 0 and i_ != args.pick:
                continue
            x = torch.randn(R, H, W, ci, device="cuda").to(torch.bfloat16)
            w = (torch.randn(co, 9, ci, device="cuda") / (9 * ci) ** 0.5).to(torch.bfloat16)
            b = torch.zeros(co, device="cuda")
            y = torch.empty(R, H, W, co, device="cuda", dtype=torch.bfloat16)
            ms = timeit(lambda: B.debug_conv3x3(x, ci, None, 0, w, None, b, None, None, y, R, H, W, co, stream=cur()),
                        args.reps)
            fl = 2.0 * R * H * W * co * 9 * ci
            tot_t += ms * cnt
            tot_f += fl * cnt
            r = dict(kind=which, shape=[R, H, W, ci, co], ms=ms, tflops=fl / ms / 1e9, frac=fl / ms / 1e9 / peak)
            out.append(r)
            print(json.dumps(r), flush=True)
        if tot_t > 0:
            print(json.dumps({which + "_weighted_tflops": tot_f / tot_t / 1e9, "frac": tot_f / tot_t / 1e9 / peak,
                              "ms_per_unit": tot_t}), flush=True)
    if args.only in ("", "gemm"):
        for i_, (M, N, K, act) in enumerate(GEMM):
            if args.pick >= 0 and i_ != args.pick:
                continue
            A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            Wt = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
            b = torch.zeros(N, device="cuda")
            D = torch.empty(M, N // 2 if act == 2 else N, device="cuda", dtype=torch.bfloat16)
            ms = timeit(lambda: B.debug_gemm(A, Wt, b, D, M, N, K, 0, act, stream=cur()), args.reps)
            fl = 2.0 * M * N * K
            r = dict(kind="gemm", shape=[M, N, K, act], ms=ms, tflops=fl / ms / 1e9, frac=fl / ms / 1e9 / peak)
            out.append(r)
            print(json.dumps(r), flush=True)


    if args.only in ("", "gemmres"):  # residual epilogues (attention out-projection, FF2, proj_out)
        for i_, (M, N, K) in enumerate([(65536, 320, 320), (65536, 320, 1280), (16384, 640, 640), (4096, 1280, 1280)]):
            if args.pick >= 0 and i_ != args.pick:
                continue
            A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            Wt = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
            b = torch.zeros(N, device="cuda")
            R = torch.randn(M, N, device="cuda").to(torch.bfloat16)
            D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            ms = timeit(lambda: B.call("sd_debug_gemm_res", B._p(A), B._p(Wt), B._p(b), B._p(R), N, B._p(D), M, N, K,
                                       B._p(cur())), args.reps)
            fl = 2.0 * M * N * K
            print(json.dumps(dict(kind="gemm_res", shape=[M, N, K], ms=ms, tflops=fl / ms / 1e9,
                                  frac=fl / ms / 1e9 / peak)), flush=True)

    if args.only in ("", "norm"):
        hbm = 6446.9
        for i_, (nb, P, C) in enumerate([(16, 4096, 320), (16, 1024, 640), (16, 256, 1280), (16, 4096, 640),
                                          (1, 262144, 128)]):
            if args.pick >= 0 and i_ != args.pick:
                continue
            x = torch.randn(nb, P, C, device="cuda").to(torch.bfloat16)
            y = torch.empty_like(x)
            gam, bet = torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")
            ms = timeit(lambda: B.call("sd_debug_groupnorm", B._p(x), B._p(y), nb, P, C, 32, B._p(gam), B._p(bet),
                                       1e-5, 1, B._p(cur())), args.reps)
            by = 3.0 * x.numel() * 2
            print(json.dumps(dict(kind="groupnorm", shape=[nb, P, C], ms=ms, gbs=by / ms / 1e6,
                                  frac=by / ms / 1e6 / hbm)), flush=True)
            ms = timeit(lambda: B.call("sd_debug_layernorm", B._p(x), B._p(y), nb * P, C, B._p(gam), B._p(bet), 1e-5,
                                       B._p(cur())), args.reps)
            by = 2.0 * x.numel() * 2
            print(json.dumps(dict(kind="layernorm", shape=[nb * P, C], ms=ms, gbs=by / ms / 1e6,
                                  frac=by / ms / 1e6 / hbm)), flush=True)
    if args.only in ("", "gnparts"):  # GroupNorm from the producers' epilogue statistics vs the 3-kernel form
        hbm = 6446.9
        for i_, (nb, P, C) in enumerate([(16, 4096, 320), (16, 1024, 640), (16, 256, 1280), (16, 4096, 640),
                                          (16, 4096, 960), (1, 262144, 128), (1, 65536, 256), (1, 16384, 512)]):
            if args.pick >= 0 and i_ != args.pick:
                continue
            x = torch.randn(nb, P, C, device="cuda").to(torch.bfloat16)
            y = torch.empty_like(x)
            gam, bet = torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")
            xs = x.double().reshape(nb, P // 32, 32, C)
            part = torch.stack([xs.sum(2), (xs * xs).sum(2)], -1).float().contiguous()
            ms3 = timeit(lambda: B.call("sd_debug_groupnorm", B._p(x), B._p(y), nb, P, C, 32, B._p(gam), B._p(bet),
                                        1e-5, 1, B._p(cur())), args.reps)
            msp = timeit(lambda: B.call("sd_debug_groupnorm_parts", B._p(x), C, B._p(part), None, 0, None, B._p(y),
                                        nb, P, 32, B._p(gam), B._p(bet), 1e-5, 1, B._p(cur())), args.reps)
            by = 2.0 * x.numel() * 2
            print(json.dumps(dict(kind="gn_parts", shape=[nb, P, C], ms_3kernel=ms3, ms_parts=msp,
                                  gbs_parts=by / msp / 1e6, frac=by / msp / 1e6 / hbm)), flush=True)
    if args.only in ("", "xattn"):  # cross-attention to 77 cached text tokens (SD-1.5 levels)
        for i_, (R, heads, d, P) in enumerate([(16, 8, 40, 4096), (16, 8, 80, 1024), (16, 8, 160, 256),
                                                (16, 8, 160, 64), (16, 10, 64, 4096), (16, 20, 64, 1024)]):
            if args.pick >= 0 and i_ != args.pick:
                continue
            C = heads * d
            q = torch.randn(R, P, C, device="cuda").to(torch.bfloat16)
            k, v = (torch.randn(R, 77, C, device="cuda").to(torch.bfloat16) for _ in range(2))
            o = torch.empty(R, P, C, device="cuda", dtype=torch.bfloat16)
            ms = timeit(lambda: B.call("sd_debug_attention", B._p(q), B._p(k), B._p(v), B._p(o), R, heads, d, P, 77,
                                       B._p(cur())), args.reps)
            by = 2.0 * q.numel() * 2
            print(json.dumps(dict(kind="xattn_mma", shape=[R, heads, d, P, 77], ms=ms, gbs=by / ms / 1e6)), flush=True)
            # the tcgen05 path: one slot per row, the engine's cache layout (K token-major, Vᵀ with 80-key slots)
            for f16 in (0, 1):
                dt = torch.float16 if f16 else torch.bfloat16
                q_ = q.to(dt).reshape(R * P, C)
                kc = torch.cat([k, v], -1).reshape(R * 77, 2 * C).to(dt).contiguous()
                vtc = torch.zeros(2 * C, R * 80, device="cuda", dtype=dt)
                for r in range(R):
                    vtc[:, r * 80:r * 80 + 77] = kc[r * 77:(r + 1) * 77].t()
                idx = torch.arange(R, device="cuda", dtype=torch.int32)
                o_ = torch.empty(R * P, C, device="cuda", dtype=dt)
                ms = timeit(lambda: B.call("sd_debug_xattention_tc", B._p(q_), B._p(kc), 2 * C, R, 0, B._p(vtc), 2 * C,
                                           R * 80, C, B._p(idx), 77, B._p(o_), R, heads, d, P, f16, B._p(cur())),
                            args.reps)
                print(json.dumps(dict(kind="xattn_tc", dtype=str(dt), shape=[R, heads, d, P, 77], ms=ms,
                                      gbs=by / ms / 1e6)), flush=True)
    if args.only in ("", "attn"):
        for i_, (R, heads, d, P) in enumerate([(16, 8, 40, 4096), (16, 8, 80, 1024), (16, 10, 64, 4096),
                                                (16, 8, 160, 256), (16, 8, 160, 64)]):
            if args.pick >= 0 and i_ != args.pick:
                continue
            C = heads * d
            qk = torch.randn(R * P, 2 * C, device="cuda").to(torch.bfloat16)
            vt = torch.randn(C, R * P, device="cuda").to(torch.bfloat16)
            o = torch.empty(R * P, C, device="cuda", dtype=torch.bfloat16)
            fl = 4.0 * R * heads * P * P * d
            for f16 in (0, 1):
                dt = torch.float16 if f16 else torch.bfloat16
                qk_, vt_ = qk.to(dt), vt.to(dt)
                o_ = torch.empty(R * P, C, device="cuda", dtype=dt)
                ms = timeit(lambda: B.call("sd_debug_attention_tc", B._p(qk_), B._p(vt_), B._p(o_), R, heads, d, P,
                                           f16, B._p(cur())), args.reps)
                print(json.dumps(dict(kind="attn_tc", dtype=str(dt), shape=[R, heads, d, P], ms=ms,
                                      tflops=fl / ms / 1e9, exp_per_s=R * heads * P * P / ms / 1e3)), flush=True)
            q, k, v = (torch.randn(R, P, C, device="cuda").to(torch.bfloat16) for _ in range(3))
            ms = timeit(lambda: B.call("sd_debug_attention", B._p(q), B._p(k), B._p(v), B._p(o), R, heads, d, P, P,
                                       B._p(cur())), args.reps)
            print(json.dumps(dict(kind="attn_mma", shape=[R, heads, d, P], ms=ms, tflops=fl / ms / 1e9)), flush=True)


if __name__ == "__main__":
    main()

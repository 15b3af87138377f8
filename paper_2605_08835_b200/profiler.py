"""Offline profiler (§III-C) on the B200.

Measures, through the engine's C ABI on two CUDA streams (UNet rounds on a high-priority stream,
VAE chunks on a low-priority stream — exactly what the GPU serving executor runs):
  τ^c(m, n, k)  concurrent latency of a stage = c rounds of (one UNet step of m requests, k of them
                without the unconditional row) ∥ (chunk ρ of each of n decodes)          (Eq. 2, R9)
  δ^c(m, n, k)  the decodes' completion: Σ_{ρ<c} round + the last round's VAE finish       (Eq. 2)
for c = 1..C_max, 0 ≤ k ≤ m ≤ B_max, 0 ≤ n ≤ m (and decode-only (0, n, 0)), in integer µs (R11).
Also: C_max by the 5 % rule and c* = argmin L(c) (Eq. 1, λ = 0.5, ties → smaller c).
Host-side orchestration only; every timed operation is a kernel of libsynerdiff.so.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import binding as B


def _rows_of(m, k):
    return 2 * m - k


class Profiler:
    def __init__(self, eng, h=64, w=64, b_max=8, reps=2, vae_sms=0):
        """vae_sms > 0: profile on the green-context SM partition the server uses with the same setting
        (sd_sm_partition_create: VAE stream on vae_sms SMs, UNet stream on the rest)."""
        self.eng, self.h, self.w, self.b_max, self.reps = eng, h, w, b_max, reps
        dev = torch.device(f"cuda:{eng.device}")
        self.part = None
        if vae_sms > 0:
            part, us, vs = C.c_void_p(), C.c_void_p(), C.c_void_p()
            nu, nv = C.c_int32(), C.c_int32()
            B.call("sd_sm_partition_create", eng.device, vae_sms, C.byref(part), C.byref(us), C.byref(vs),
                   C.byref(nu), C.byref(nv))
            self.part, self.partition_sms = part, (nu.value, nv.value)
            self.hi = torch.cuda.ExternalStream(us.value, device=dev)
            self.lo = torch.cuda.ExternalStream(vs.value, device=dev)
        else:
            self.hi = torch.cuda.Stream(device=dev, priority=-1)
            self.lo = torch.cuda.Stream(device=dev, priority=0)
        g = torch.Generator(device="cpu").manual_seed(0)
        self.lat = [torch.randn(4, h, w, generator=g).to(dev) for _ in range(b_max)]
        self.lat_save = [t.clone() for t in self.lat]
        self.dec = [torch.randn(4, h, w, generator=g).to(dev) for _ in range(b_max)]
        self.img = [torch.empty(3, eng.upscale * h, eng.upscale * w, device=dev) for _ in range(b_max)]
        emb = torch.randn(eng.ctx_len, eng.ctx_dim, generator=g)
        pooled = torch.randn(eng.pooled_dim, generator=g) if eng.pooled_dim else None  # SDXL added conditioning
        self.slots = [eng.register(emb, pooled) for _ in range(b_max)]

    def close(self):
        for s in self.slots:
            self.eng.release(s)
        if self.part is not None:
            torch.cuda.synchronize()
            B.call("sd_sm_partition_destroy", self.part)
            self.part = None

    def _stage(self, c, m, n, k):
        """One stage (m, n, k) at granularity c; returns (τ µs, δ µs)."""
        eng = self.eng
        states = [C.c_void_p() for _ in range(n)]
        tau = 0.0
        delta = 0.0
        for rho in range(c):
            e0 = torch.cuda.Event(enable_timing=True)
            eh, el = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.hi)
            self.lo.wait_event(e0)
            if m:
                eng.step(self.lat[:m], [10] * m, [50] * m, [0] * k + [1] * (m - k), [7.5] * m, self.slots[:m],
                         stream=self.hi)
            for i in range(n):
                eng.decode_chunk(self.dec[i], c, rho, states[i], self.img[i], stream=self.lo)
            eh.record(self.hi)
            el.record(self.lo)
            eh.synchronize()
            el.synchronize()
            th = e0.elapsed_time(eh) * 1e3 if m else 0.0
            tl = e0.elapsed_time(el) * 1e3 if n else 0.0
            r = max(th, tl)
            if rho == c - 1:
                delta = tau + tl
            tau += r
        for i in range(m):
            self.lat[i].copy_(self.lat_save[i])
        return int(round(tau)), (int(round(delta)) if n else 0)

    def measure(self, c_values, b_max=None, n_max=None, progress=None):
        """Full τ/δ table {(c, m, n, k): (tau_us, delta_us)} (median of `reps` measurements)."""
        b_max = b_max or self.b_max
        n_max = b_max if n_max is None else n_max
        tab = {}
        keys = []
        for c in c_values:
            for m in range(0, b_max + 1):
                for n in range(0, n_max + 1):
                    for k in range(0, m + 1):
                        if (m == 0 and n == 0) or (m >= 1 and n > m) or (m == 0 and k):
                            continue
                        if c > 1 and n == 0:
                            continue  # pure-UNet windows always run one round (R8): only c = 1 needed
                        keys.append((c, m, n, k))
        # warm every (rows) graph and decode slot once
        for key in keys[: min(len(keys), 12)]:
            self._stage(*key)
        for key in keys:
            vals = sorted(self._stage(*key) for _ in range(self.reps))
            tab[key] = vals[len(vals) // 2]
            if progress:
                progress(key, tab[key])
        for c in c_values:                       # τ^c(m,0,k) := c · τ^1(m,0,k) (pure rounds, Eq. 2 with n = 0)
            if c > 1:
                for (cc, m, n, k), v in list(tab.items()):
                    if cc == 1 and n == 0:
                        tab[(c, m, 0, k)] = (c * v[0], 0)
        return tab


def to_table_handle(tab):
    keys = sorted(tab)
    n = len(keys)
    col = lambda i: (C.c_int32 * n)(*[k[i] for k in keys])
    h = C.c_void_p()
    B.call("sd_table_from_arrays", n, col(0), col(1), col(2), col(3), (C.c_int64 * n)(*[tab[k][0] for k in keys]),
           (C.c_int64 * n)(*[tab[k][1] for k in keys]), C.byref(h))
    return h


def write_csv(tab, path):
    with open(path, "w") as f:
        f.write("c,m,n,k,tau_us,delta_us\n")
        for k in sorted(tab):
            f.write(f"{k[0]},{k[1]},{k[2]},{k[3]},{tab[k][0]},{tab[k][1]}\n")


def chunk_choice(tab, c_values, m, n=1, lam=(1, 2)):
    """C_max (5 % rule) and c* = argmin Eq. 1 L(c) at (m, n, 0) against solo baselines —
    computed by sd_chunk_choice in libsynerdiff.so (exact rationals); lam = λ as (num, den), paper 0.5."""
    h = to_table_handle(tab)
    try:
        k = len(c_values)
        cmax, cstar, cost = C.c_int32(), C.c_int32(), (C.c_double * k)()
        B.call("sd_chunk_choice", h, m, n, (C.c_int32 * k)(*c_values), k, lam[0], lam[1], C.byref(cmax),
               C.byref(cstar), cost)
    finally:
        B.lib().sd_table_free(h)
    return cmax.value, cstar.value, {c: cost[i] for i, c in enumerate(c_values)}


def solo_unet_table(prof, m_max, reps=3):
    """τ^1(m, 0, 0) for m = 1 … m_max (one UNet step of m requests with CFG, no decode), µs: the input of
    the B_max saturation rule."""
    tab = {}
    for m in range(1, m_max + 1):
        vals = sorted(prof._stage(1, m, 0, 0)[0] for _ in range(reps))
        tab[(1, m, 0, 0)] = (vals[len(vals) // 2], 0)
    return tab


def find_b_max(tab, m_max, eps=(1, 20)):
    """B_max by sd_find_b_max on a table holding (1, m, 0, 0) for m = 1 … m_max."""
    h = to_table_handle(tab)
    try:
        out = C.c_int32()
        B.call("sd_find_b_max", h, m_max, eps[0], eps[1], C.byref(out))
    finally:
        B.lib().sd_table_free(h)
    return out.value

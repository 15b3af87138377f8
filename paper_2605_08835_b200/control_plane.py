"""C1, the control-plane collective of the multi-GPU path (PAPER.md:307 the
controller "monitors queue trends"): every rank periodically all-gathers its serving loop's load
int32[4] = {waiting, decode-pending, active, completed} and hands the [P][4] snapshot to
sd_set_global_load, so every rank's controller sees the summed waiting queue (R15).

It runs on its own thread, its own process group (communicator) and — for NCCL — its own CUDA stream,
so the data plane (sd_step_batch / VAE chunks on the serving loop's streams) never waits on a peer.
A fifth int per rank is a done flag: the loop ends after the collective in which every rank reported
done, so every rank issues the same number of collectives. Marshalling only: the loads come from and
go back into libsynerdiff.so; the collective is torch.distributed (NCCL on GPUs, gloo in the tests).
"""
from __future__ import annotations

import ctypes as C
import threading
import time

import torch
import torch.distributed as dist

from . import binding as B


class LoadGather:
    """`source` is an engine (sd_get_load / sd_set_global_load) or any object with get_load() -> 4 ints and
    set_global(list of 4·P ints, P, epoch). device=None → CPU tensors (gloo); an int → that CUDA device
    (NCCL), with a private stream."""

    def __init__(self, source, world, rank, group=None, device=None, period_s=0.05):
        self.src, self.world, self.rank, self.group = source, world, rank, group
        self.device = device
        self.period = period_s
        self._stop = threading.Event()
        self._th = None
        self.epochs = 0
        self.times_us = []
        self.snapshots = []

    def _get(self):
        if hasattr(self.src, "get_load"):
            return list(self.src.get_load())
        v = (C.c_int32 * 4)()
        B.call("sd_get_load", self.src.h, v)
        return list(v)

    def _set(self, flat, epoch):
        if hasattr(self.src, "set_global"):
            return self.src.set_global(flat, self.world, epoch)
        B.call("sd_set_global_load", self.src.h, (C.c_int32 * len(flat))(*flat), self.world, epoch)

    def exchange(self, done: bool):
        """One collective: returns (flat [P][4] loads, all_done)."""
        dev = "cpu" if self.device is None else f"cuda:{self.device}"
        mine = torch.tensor(self._get() + [1 if done else 0], dtype=torch.int32, device=dev)
        allv = torch.zeros(5 * self.world, dtype=torch.int32, device=dev)
        t0 = time.perf_counter()
        dist.all_gather_into_tensor(allv, mine, group=self.group)
        v = allv.cpu().tolist()
        self.times_us.append((time.perf_counter() - t0) * 1e6)
        flat = [x for r in range(self.world) for x in v[5 * r:5 * r + 4]]
        return flat, all(v[5 * r + 4] for r in range(self.world))

    def _loop(self):
        stream = torch.cuda.Stream(device=self.device) if self.device is not None else None
        ctx = torch.cuda.stream(stream) if stream is not None else _Null()
        with ctx:
            while True:
                flat, all_done = self.exchange(self._stop.is_set())
                if all_done:
                    break
                self._set(flat, self.epochs)
                self.snapshots.append(flat)
                self.epochs += 1
                time.sleep(self.period)

    def start(self):
        self._th = threading.Thread(target=self._loop, daemon=True)
        self._th.start()

    def stop(self, timeout_s=600):
        self._stop.set()
        if self._th:
            self._th.join(timeout=timeout_s)

    def mean_us(self):
        return sum(self.times_us) / len(self.times_us) if self.times_us else None


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False

"""Multi-GPU host logic on CPU: world_size 2 over gloo.

Each rank serves the shard {id : id mod P = rank}; the only collective is the all-gather of the
per-rank loads int32[4] = {waiting, decode-pending, active, completed}; every rank feeds the summed
waiting queue to its controller, so all ranks take identical directives (bit-exact)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import ctypes as C

    from paper_2605_08835_b200 import binding as B
    from paper_2605_08835_b200.serving import poisson_trace
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # sharding: every rank generates the whole trace from the shared seed and keeps id mod P
    trace = poisson_trace(64, 5.0, seed=3)
    mine = [t for t in trace if t[0] % world == rank]
    # controller fed by the all-gathered loads
    cfg = B.ControllerConfig(1, 4, 10, 3, 1, 2, -1, 5)
    h = C.c_void_p()
    B.call("sd_controller_create", C.byref(cfg), C.byref(h))
    rng = np.random.default_rng(100 + rank)
    q_local, traj, gathered_log = 0, [], []
    for step in range(200):
        q_local = max(0, q_local + int(rng.integers(-1, 3 if step < 90 else 1)))
        loads = torch.tensor([q_local, rank, 8, step], dtype=torch.int32)
        allv = [torch.zeros(4, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(allv, loads)
        glob = int(sum(int(v[0]) for v in allv))
        d = B.Directive()
        B.call("sd_controller_decide", h, step * 100_000, glob, C.byref(d))
        traj.append((d.level, d.c))
        gathered_log.append([int(v[1]) for v in allv])
    B.lib().sd_controller_free(h)
    q.put((rank, [t[0] for t in mine], traj, gathered_log))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_allgather_controller_and_sharding():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, ids, traj, glog = q.get(timeout=240)
        res[r] = (ids, traj, glog)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids0, ids1 = res[0][0], res[1][0]
    assert not set(ids0) & set(ids1) and sorted(ids0 + ids1) == list(range(64))      # a partition
    assert all(i % 2 == 0 for i in ids0) and all(i % 2 == 1 for i in ids1)
    assert res[0][1] == res[1][1]                        # identical directives on every rank
    assert all(g == [0, 1] for g in res[0][2])           # all-gather is rank-ordered
    assert max(t[0] for t in res[0][1]) >= 1             # the summed queue drove escalation


class _VServe:
    """Adapter: a stepping virtual-clock server (sd_vserve_*) as LoadGather's load source."""

    def __init__(self, h):
        self.h = h

    def get_load(self):
        import ctypes as C

        from paper_2605_08835_b200 import binding as B
        v = (C.c_int32 * 4)()
        B.call("sd_vserve_get_load", self.h, v)
        return list(v)

    def set_global(self, flat, P, epoch):
        import ctypes as C

        from paper_2605_08835_b200 import binding as B
        B.call("sd_vserve_set_global_load", self.h, (C.c_int32 * len(flat))(*flat), P, epoch)


def _serve_worker(rank, world, port, q):
    """One rank of SURVEY §8(e) on the virtual clock: this rank's shard {id mod P = rank} served by the C++
    loop (sd_vserve_*), one window per epoch, the C1 all-gather (control_plane.LoadGather over gloo)
    between epochs feeding sd_vserve_set_global_load."""
    import ctypes as C
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_cabi_host import make_multi_table, serve_table

    from paper_2605_08835_b200 import binding as B
    from paper_2605_08835_b200.control_plane import LoadGather
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tabs = serve_table(np.random.default_rng(5))
    h = make_multi_table(tabs)
    trace = _sharded_trace()
    mine = [e for e in trace if e[0] % world == rank]
    n = len(mine)
    ctl = B.ControllerConfig(1, 4, 10, 3, 1, 2, -1, 5)
    cfg = B.ServeConfig(8, 1, 10, 0, 1, ctl, h, 64, 1)
    v = C.c_void_p()
    B.call("sd_vserve_create", C.byref(cfg), h, n, (C.c_uint64 * n)(*[e[0] for e in mine]),
           (C.c_int64 * n)(*[e[1] for e in mine]), (C.c_int32 * n)(*[e[2] for e in mine]), C.byref(v))
    lg = LoadGather(_VServe(v), world, rank, device=None)
    st = C.c_int32()
    epochs = 0
    while True:
        B.call("sd_vserve_window", v, C.byref(st))
        flat, all_done = lg.exchange(st.value == -1)
        if all_done:
            break
        lg._set(flat, epochs)
        epochs += 1
    U, V = (C.c_int64 * n)(), (C.c_int64 * n)()
    ns, win, now = (C.c_int32 * n)(), C.c_int32(), C.c_int64()
    B.call("sd_vserve_results", v, U, V, ns, C.byref(now), C.byref(win))
    cap = 1 << 14
    w, la, ca, nt = (C.c_int32 * cap)(), (C.c_int32 * cap)(), (C.c_int32 * cap)(), C.c_int32()
    B.call("sd_vserve_trajectory", v, cap, w, la, ca, C.byref(nt))
    traj = [(w[i], la[i], ca[i]) for i in range(nt.value)]
    B.lib().sd_vserve_free(v)
    B.lib().sd_table_free(h)
    q.put((rank, [e[0] for e in mine], list(U), list(V), list(ns), traj, epochs))
    dist.destroy_process_group()


def _sharded_trace():
    rng = np.random.default_rng(77)
    n = 160
    arr = np.cumsum(rng.exponential(1e6 / 14.0, n)).astype(np.int64)
    steps = rng.integers(20, 51, n)
    return [(i, int(arr[i]), int(steps[i])) for i in range(n)]


@pytest.mark.timeout(300)
def test_two_rank_sharded_serving_bitexact_vs_oracle():
    """world_size 2 over gloo: each rank serves its shard with the C++ loop (virtual clock) and the C1
    all-gather of loads between windows; every request's (U, V, #skips) and every window's (waiting
    observed, level, c) equal oracle/serving.simulate_sharded (lockstep epochs, the same snapshot rule)
    bit for bit — and the summed-queue controller engages Skip-CFG."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_cabi_host import serve_table

    from oracle import serving
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_serve_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=240)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tabs = serve_table(np.random.default_rng(5))
    done, logs = serving.simulate_sharded(_sharded_trace(), world, tabs, c_star=1, c_max=4)
    assert res[0][5] == res[1][5]                     # both ranks ran the same number of epochs
    skips = 0
    for r in range(world):
        ids, U, V, ns, traj, _ = res[r]
        assert sorted(done[r]) == sorted(ids)
        for j, i in enumerate(ids):
            t = done[r][i]
            assert (U[j], V[j], ns[j]) == (t.U, t.V, len(t.skips)), (r, i)
        assert traj == [(w["waiting"], w["level_after"], w["c_after"]) for w in logs[r]], r
        skips += sum(ns)
    assert skips > 0
    # the exchange matters: serving each shard on its own (controller on the local queue) gives a
    # different timeline for many requests
    alone = [serving.simulate([e for e in _sharded_trace() if e[0] % world == r], tabs, b_max=8, c_star=1, c_max=4)
             for r in range(world)]
    assert sum((alone[r][i].U, alone[r][i].V) != (done[r][i].U, done[r][i].V) for r in range(world)
               for i in done[r]) > 10

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

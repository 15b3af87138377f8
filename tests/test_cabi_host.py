"""CPU tests of libsynerdiff.so: it loads, exports every symbol include/sd_api.h declares, and its
host control plane (latency table, Problem P planner, controller, VAE chunk partition) makes the
same decisions as the independent oracle, bit-exactly (north star: "scheduler decisions bit-exact")."""
import ctypes as C
import os
import re
import tempfile

import numpy as np
import pytest

from oracle import controller as octl
from oracle import sched, vae
from paper_2605_08835_b200 import binding as B

HDR = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "sd_api.h")


def declared_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:sd_status|const char\*)\s+(sd_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    L = B.lib()
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
        assert n in B.SIGNATURES, n


def test_status_strings_and_validation():
    assert B.status_str(B.SD_E_CUDA) == "SD_E_CUDA"
    # invalid arguments are rejected before any work (no GPU needed)
    st = B.lib().sd_plan(None, 1, 1, 0, 1, 1, 10, 0, None, 0, None, None, None)
    assert st == B.SD_E_INVAL and "sd_plan" in B.last_error()
    h = C.c_void_p()
    cfg = B.EngineConfig(7, 0, 0, 64, 8, 16, 0)
    assert B.lib().sd_engine_create(C.byref(cfg), 0, C.byref(h)) == B.SD_E_INVAL


def make_table(tab, c=1):
    keys = sorted(tab)
    n = len(keys)
    arr = lambda xs, t: (t * n)(*xs)
    h = C.c_void_p()
    B.call("sd_table_from_arrays", n, arr([c] * n, C.c_int32), arr([k[0] for k in keys], C.c_int32),
           arr([k[1] for k in keys], C.c_int32), arr([k[2] for k in keys], C.c_int32),
           arr([tab[k][0] for k in keys], C.c_int64), arr([tab[k][1] for k in keys], C.c_int64), C.byref(h))
    return h


def cplan(h, M, N, K, a_num=1, a_den=10, mode=0, c=1):
    out = (C.c_int32 * 300)()
    ns, cost, tm = C.c_int32(), C.c_int64(), C.c_int64()
    B.call("sd_plan", h, M, N, K, c, a_num, a_den, mode, out, 100, C.byref(ns), C.byref(cost), C.byref(tm))
    return tuple(tuple(out[3 * i:3 * i + 3]) for i in range(ns.value)), cost.value, tm.value


def random_table(rng, B_=6):
    tab = {}
    for m in range(0, B_ + 1):
        for n in range(0, B_ + 1):
            for k in range(0, m + 1):
                if m == 0 and n == 0:
                    continue
                tau = int(round((5 + 20 * max(m - 0.5 * k, 0) ** 0.8 + 15 * n + int(rng.integers(0, 9))) * 1000))
                tab[(m, n, k)] = (tau, int(round(tau * rng.uniform(0.4, 1.0))) if n else 0)
    return tab


def test_plan_bitexact_vs_oracle():
    rng = np.random.default_rng(11)
    n = 0
    for trial in range(10):
        tab = random_table(rng, 6)
        h = make_table(tab)
        for M in range(0, 7):
            for N in range(0, 7):
                for K in range(0, M + 1):
                    for a_num, a_den in ((1, 10), (10, 1)):
                        for mode in (0, 1):
                            got = cplan(h, M, N, K, a_num, a_den, mode)
                            exp = sched.plan_window(tab, M, N, K, a_num, a_den, "exact" if mode == 0 else "alg1")
                            assert got[0] == tuple(exp), (M, N, K, mode, got, exp)
                            assert (got[1], got[2]) == sched.plan_cost(tab, exp) if exp else True
                            n += 1
        B.lib().sd_table_free(h)
    assert n > 2000


def test_plan_speed_8x8x8():
    import time
    rng = np.random.default_rng(3)
    tab = random_table(rng, 8)
    h = make_table(tab)
    t0 = time.perf_counter()
    for _ in range(20):
        cplan(h, 8, 8, 8)
    dt = (time.perf_counter() - t0) / 20
    assert dt < 0.05          # SPEC acceptance 9: < 50 ms ("millisecond-level")


def test_table_csv_roundtrip_and_errors():
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.csv")
        open(p, "w").write("c,m,n,k,tau_us,delta_us\n1,1,1,0,46300,20800\n1,1,0,0,40000,0\n")
        h = C.c_void_p()
        B.call("sd_table_load", p.encode(), C.byref(h))
        assert cplan(h, 1, 1, 0)[0] == ((1, 1, 0),)
        open(p, "w").write("c,m,n,k,tau_us,delta_us\n1,1,1,0,46300,20800\n1,1,1,0,1,1\n")
        assert B.lib().sd_table_load(p.encode(), C.byref(h)) == B.SD_E_INVAL
        assert "duplicate" in B.last_error()
        open(p, "w").write("c,m,n,k,tau_us,delta_us\n1,1,x,0,46300,20800\n")
        assert B.lib().sd_table_load(p.encode(), C.byref(h)) == B.SD_E_INVAL


def test_plan_table_miss_is_an_error():
    h = make_table({(1, 1, 0): (10, 5)})
    out = (C.c_int32 * 30)()
    ns = C.c_int32()
    st = B.lib().sd_plan(h, 2, 1, 0, 1, 1, 10, 0, out, 10, C.byref(ns), None, None)
    assert st == B.SD_E_INVAL and "table miss" in B.last_error()


@pytest.mark.parametrize("pulse", [1, 2])
def test_controller_bitexact_vs_oracle(pulse):
    cfg = B.ControllerConfig(1, 4, 10, 3, 1, 2, -1, 5)
    h = C.c_void_p()
    B.call("sd_controller_create", C.byref(cfg), C.byref(h))
    ref = octl.Controller(c_star=1, c_max=4, window=10, h=3)
    rng = np.random.default_rng(pulse)
    q, t = 0, 0
    traj = []
    for i in range(600):
        t += int(rng.integers(50_000, 400_000))
        q = max(0, q + int(rng.integers(-2, 4 if i < 250 else 1)))
        d = B.Directive()
        B.call("sd_controller_decide", h, t, q, C.byref(d))
        lv, c, ch = ref.decide(t, q)
        assert (d.level, d.c, bool(d.changed)) == (lv, c, ch), i
        traj.append((lv, c))
    assert max(x[0] for x in traj) == 2
    B.lib().sd_controller_free(h)


def test_chunk_ranges_bitexact_vs_oracle():
    rng = np.random.default_rng(8)
    for _ in range(300):
        n = int(rng.integers(1, 40))
        c = int(rng.integers(1, 17))
        costs = [int(x) for x in rng.integers(0 if _ % 3 else 1, 1000, n)]
        costs = [max(1, x) for x in costs]
        out = (C.c_int32 * (c + 2))()
        B.call("sd_chunk_ranges", (C.c_int64 * n)(*costs), n, c, out)
        exp = vae.chunk_ranges(costs, c)
        assert list(out[:len(exp)]) == exp


# ---- serving loop, virtual clock (T5/T6: decisions and timestamps bit-exact with oracle/serving.py) ----

def serve_table(rng, B_=8, cmax=4):
    """τ^c/δ^c per (c, m, n, k): Eq. 2 composition of a synthetic per-round model (µs)."""
    tabs = {}
    for c in range(1, cmax + 1):
        t = {}
        for m in range(0, B_ + 1):
            for n in range(0, B_ + 1):
                for k in range(0, m + 1):
                    if m == 0 and n == 0:
                        continue
                    if m >= 1 and n > m:
                        continue
                    if m == 0 and k:
                        continue
                    tu = int(8000 + 2500 * (2 * m - k)) if m else 0
                    tv = (int(60000 * n / c) + 3000) if n else 0
                    rounds_u = [tu] * c
                    rounds_v = [tv] * c
                    Tu, Tv = sched.cumulative_latencies(rounds_u, rounds_v) if n else (sum(rounds_u), 0)
                    t[(m, n, k)] = (Tu, Tv if n else 0)
        tabs[c] = t
    return tabs


def make_multi_table(tabs):
    keys = [(c, *k) for c in sorted(tabs) for k in sorted(tabs[c])]
    n = len(keys)
    h = C.c_void_p()
    col = lambda i, t: (t * n)(*[k[i] for k in keys])
    B.call("sd_table_from_arrays", n, col(0, C.c_int32), col(1, C.c_int32), col(2, C.c_int32), col(3, C.c_int32),
           (C.c_int64 * n)(*[tabs[k[0]][k[1:]][0] for k in keys]),
           (C.c_int64 * n)(*[tabs[k[0]][k[1:]][1] for k in keys]), C.byref(h))
    return h


@pytest.mark.parametrize("rate,mode,cstar", [(2.0, 0, 1), (6.0, 0, 1), (6.0, 1, 2), (12.0, 0, 1)])
def test_serving_simulation_bitexact(rate, mode, cstar):
    from oracle import serving
    rng = np.random.default_rng(int(rate * 10) + mode)
    tabs = serve_table(rng)
    h = make_multi_table(tabs)
    n = 120
    gaps = rng.exponential(1e6 / rate, n)
    arr = np.cumsum(gaps).astype(np.int64)
    steps = rng.integers(20, 51, n)
    trace = [(i, int(arr[i]), int(steps[i])) for i in range(n)]
    ctl_cfg = B.ControllerConfig(cstar, 4, 10, 3, 1, 2, -1, 5)
    cfg = B.ServeConfig(8, 1, 10, mode, cstar, ctl_cfg, h, 64, 1)
    U, V = (C.c_int64 * n)(), (C.c_int64 * n)()
    ns, win = (C.c_int32 * n)(), C.c_int32()
    B.call("sd_serve_simulate", C.byref(cfg), h, n, (C.c_uint64 * n)(*range(n)), (C.c_int64 * n)(*arr.tolist()),
           (C.c_int32 * n)(*steps.tolist()), U, V, ns, C.byref(win))
    log = []
    done = serving.simulate(trace, tabs, b_max=8, mode="exact" if mode == 0 else "alg1", c_star=cstar, c_max=4,
                            log=log)
    assert len(done) == n and win.value == len(log)
    for i in range(n):
        t = done[i]
        assert (U[i], V[i], ns[i]) == (t.U, t.V, len(t.skips)), i
        assert t.A <= t.U <= t.V
        # skip audit: every skipped step index respects the most permissive s_min (⌈0.5 n⌉)
        assert all(s >= (t.n + 1) // 2 for s in t.skips)
    m = serving.metrics(done)
    assert m["p99_e2e_us"] >= m["mean_e2e_us"] * 0.5
    if rate >= 12:
        assert any(w["level"] > 0 for w in log) and sum(ns) > 0     # the controller engaged Skip-CFG
    B.lib().sd_table_free(h)


@pytest.mark.parametrize("policy,ablation,cstar,cmax", [("serial", 0, 1, 1), ("dynamic", 0, 1, 1), ("naive", 0, 2, 4),
                                                         ("synerdiff", 1, 1, 4), ("synerdiff", 2, 2, 4),
                                                         ("synerdiff", 0, 1, 1)])
def test_serving_policies_bitexact(policy, ablation, cstar, cmax):
    """Baselines and ablations: the C++ loop on the virtual clock equals
    oracle/serving.py for every request's (U, V, #skips) and the number of windows."""
    from oracle import serving
    rng = np.random.default_rng(len(policy) * 7 + ablation)
    tabs = serve_table(rng)
    h = make_multi_table(tabs)
    n = 90
    gaps = rng.exponential(1e6 / 8.0, n)
    arr = np.cumsum(gaps).astype(np.int64)
    steps = rng.integers(20, 51, n)
    trace = [(i, int(arr[i]), int(steps[i])) for i in range(n)]
    ctl_cfg = B.ControllerConfig(cstar, cmax, 10, 3, 1, 2, -1, 5)
    cfg = B.ServeConfig(8, 1, 10, 0, cstar, ctl_cfg, h, 64, 1, 4, B.POLICIES[policy], ablation, 300_000)
    U, V = (C.c_int64 * n)(), (C.c_int64 * n)()
    ns, win = (C.c_int32 * n)(), C.c_int32()
    B.call("sd_serve_simulate", C.byref(cfg), h, n, (C.c_uint64 * n)(*range(n)), (C.c_int64 * n)(*arr.tolist()),
           (C.c_int32 * n)(*steps.tolist()), U, V, ns, C.byref(win))
    done = serving.simulate(trace, tabs, b_max=8, c_star=cstar, c_max=cmax, policy=policy,
                            no_skip=bool(ablation & B.SD_ABL_NO_SKIP), no_ctl=bool(ablation & B.SD_ABL_NO_CTL),
                            dyn_window_us=300_000, n_max=4)
    assert len(done) == n
    for i in range(n):
        t = done[i]
        assert (U[i], V[i], ns[i]) == (t.U, t.V, len(t.skips)), (policy, i)
    if ablation & B.SD_ABL_NO_SKIP or policy != "synerdiff":
        assert sum(ns) == 0
    B.lib().sd_table_free(h)


@pytest.mark.parametrize("policy", ["synerdiff", "naive", "dynamic", "serial"])
def test_serving_mixed_resolution_bitexact(policy):
    """Mixed-resolution traces: the C++ loop with per-resolution tables equals
    oracle/serving.py (largest-resolution table per window) for every request's (U, V, #skips)."""
    from oracle import serving
    rng = np.random.default_rng(31 + len(policy))
    tabs = {64: serve_table(rng), 96: serve_table(rng)}
    for r in tabs[96]:  # the 768² table is slower
        tabs[96][r] = {k: (2 * v[0] + 100, 2 * v[1] + 50) for k, v in tabs[96][r].items()}
    handles = {r: make_multi_table(t) for r, t in tabs.items()}
    n = 80
    arr = np.cumsum(rng.exponential(1e6 / 6.0, n)).astype(np.int64)
    steps = rng.integers(20, 51, n)
    res = rng.choice([64, 96], n)
    ctl_cfg = B.ControllerConfig(1, 4, 10, 3, 1, 2, -1, 5)
    hw = (C.c_int32 * 2)(64, 96)
    tbl = (C.c_void_p * 2)(handles[64].value, handles[96].value)
    cfg = B.ServeConfig(8, 1, 10, 0, 1, ctl_cfg, None, 64, 1, 4, B.POLICIES[policy], 0, 300_000, 2,
                        C.cast(hw, C.POINTER(C.c_int32)), C.cast(tbl, C.POINTER(C.c_void_p)))
    U, V = (C.c_int64 * n)(), (C.c_int64 * n)()
    ns, win = (C.c_int32 * n)(), C.c_int32()
    B.call("sd_serve_simulate_mixed", C.byref(cfg), n, (C.c_uint64 * n)(*range(n)), (C.c_int64 * n)(*arr.tolist()),
           (C.c_int32 * n)(*steps.tolist()), (C.c_int32 * n)(*res.tolist()), U, V, ns, C.byref(win))
    trace = [(i, int(arr[i]), int(steps[i]), int(res[i])) for i in range(n)]
    done = serving.simulate(trace, None, b_max=8, c_star=1, c_max=4, policy=policy, dyn_window_us=300_000, n_max=4,
                            res_tables=tabs)
    for i in range(n):
        t = done[i]
        assert (U[i], V[i], ns[i]) == (t.U, t.V, len(t.skips)), (policy, i)
    for h in handles.values():
        B.lib().sd_table_free(h)


def test_plan_alg1_hand_trace():
    """sd_plan in both modes on the hand-traced Alg. 1 window (tests/golden/alg1_trace.json)."""
    import json
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "alg1_trace.json")))
    tab = {tuple(e["mnk"]): (e["tau"], e["delta"]) for e in g["table"]}
    h = make_table(tab)
    w = g["window"]
    for mode, key in ((1, "alg1_result"), (0, "exact_result")):
        st, cost, tm = cplan(h, w["M"], w["N"], w["K"], mode=mode)
        r = g[key]
        assert (st, cost, tm) == (tuple(tuple(s) for s in r["stages"]), r["cost"], r["time"]), key
    B.lib().sd_table_free(h)


def test_map_tasks_bitexact_vs_oracle():
    """Task mapping E (R14): sd_map_tasks equals oracle.sched.map_tasks on random windows."""
    rng = np.random.default_rng(11)
    tab = random_table(rng)
    checked = 0
    for trial in range(300):
        M = int(rng.integers(1, 7))
        N = int(rng.integers(0, M + 1))
        ns_ = rng.integers(2, 40, M)
        ss = [int(rng.integers(0, n)) for n in ns_]
        elig = [int(rng.random() < 0.6) for _ in range(M)]
        K = sum(elig)
        ids = [int(x) for x in rng.permutation(100)[:M]]
        dids = [int(x) for x in rng.permutation(100)[:N]]
        darr = [int(x) for x in rng.integers(0, 5, N)]                       # ties on A → id decides
        stages = sched.plan_window(tab, M, N, K) if N else ((M, 0, 0),)
        E = sched.map_tasks(stages, [(ids[i], ss[i], int(ns_[i]), bool(elig[i])) for i in range(M)],
                            [(dids[j], darr[j]) for j in range(N)])
        want_u = {}
        want_d = {}
        for t, (u_ids, skip_ids, d_ids) in enumerate(E):
            for x in u_ids:
                want_u[x] = (t, int(x in skip_ids))
            for x in d_ids:
                want_d[x] = t
        T = len(stages)
        us, sk, ds = (C.c_int32 * M)(), (C.c_uint8 * M)(), (C.c_int32 * max(N, 1))()
        B.call("sd_map_tasks", (C.c_int32 * (3 * T))(*[v for s in stages for v in s]), T, M,
               (C.c_uint64 * M)(*ids), (C.c_int32 * M)(*ss), (C.c_int32 * M)(*[int(x) for x in ns_]),
               (C.c_uint8 * M)(*elig), N, (C.c_uint64 * max(N, 1))(*dids), (C.c_int64 * max(N, 1))(*darr),
               us, sk, ds)
        assert [(us[i], sk[i]) for i in range(M)] == [want_u[x] for x in ids]
        assert [ds[j] for j in range(N)] == [want_d[x] for x in dids]
        checked += 1
    assert checked == 300
    bad = B.lib().sd_map_tasks((C.c_int32 * 3)(2, 0, 0), 1, 1, (C.c_uint64 * 1)(0), (C.c_int32 * 1)(0),
                               (C.c_int32 * 1)(5), (C.c_uint8 * 1)(0), 0, None, None, (C.c_int32 * 1)(),
                               (C.c_uint8 * 1)(), None)
    assert bad == B.SD_E_INVAL


@pytest.mark.parametrize("mode", [0, 1])
def test_vserve_decision_replay(mode):
    """T5 on the virtual clock: every window's logged decision (stages S and mapping E) is recomputed from
    the logged window inputs by oracle.sched.plan_window and oracle.sched.map_tasks and must be equal bit
    for bit."""
    from oracle import sched as osched
    rng = np.random.default_rng(5 + mode)
    tabs = serve_table(rng)
    h = make_multi_table(tabs)
    n = 150
    arr = np.cumsum(rng.exponential(1e6 / 9.0, n)).astype(np.int64)
    steps = rng.integers(20, 51, n)
    ctl_cfg = B.ControllerConfig(1, 4, 10, 3, 1, 2, -1, 5)
    cfg = B.ServeConfig(8, 1, 10, mode, 1, ctl_cfg, h, 64, 1)
    v = C.c_void_p()
    B.call("sd_vserve_create", C.byref(cfg), h, n, (C.c_uint64 * n)(*range(n)), (C.c_int64 * n)(*arr.tolist()),
           (C.c_int32 * n)(*steps.tolist()), C.byref(v))
    state = C.c_int32()
    windows = 0
    while True:
        B.call("sd_vserve_window", v, C.byref(state))
        if state.value < 0:
            break
        windows += state.value
    assert windows > 100
    n_skipping = n_chunked = 0
    for w in range(windows):
        level, c, stages, unet, dec = B.window_plan("sd_vserve_window_plan", v, w)
        M, N = len(unet), len(dec)
        K = sum(u[3] for u in unet)
        smin = {0: None, 1: lambda n_: -(-7 * n_ // 10), 2: lambda n_: -(-n_ // 2)}[level]
        assert [u[3] for u in unet] == [int(smin is not None and u[1] >= smin(u[2])) for u in unet]   # R6
        want = osched.plan_window(tabs[c], M, N, K, mode="exact" if mode == 0 else "alg1")
        assert stages == want, (w, M, N, K, c, stages, want)
        E = osched.map_tasks(stages, [(u[0], u[1], u[2], bool(u[3])) for u in unet], [(d[0], d[1]) for d in dec])
        got_u = {u[0]: (u[4], u[5]) for u in unet}
        got_d = {d[0]: d[2] for d in dec}
        for t, (u_ids, skip_ids, d_ids) in enumerate(E):
            for x in u_ids:
                assert got_u[x] == (t, int(x in skip_ids)), (w, x)
            for x in d_ids:
                assert got_d[x] == t, (w, x)
        n_skipping += sum(s[2] for s in stages) > 0
        n_chunked += c > 1 and N > 0
    assert n_skipping > 0 and n_chunked > 0     # the trace exercises Skip-CFG slots and c > 1 plans
    B.lib().sd_vserve_free(v)
    B.lib().sd_table_free(h)


def test_chunk_choice_bitexact_vs_oracle():
    """sd_chunk_choice (Eq. 1 L(c), c* = argmin with ties to the smaller c, and the C_max 5 % rule of
    PAPER.md:248; R31) equals oracle.sched.chunk_cost / select_c / find_c_max evaluated in exact Fractions
    on random profiled tables, including constructed exact ties."""
    from fractions import Fraction as F
    from paper_2605_08835_b200 import profiler
    rng = np.random.default_rng(3)
    for trial in range(200):
        cs = [1, 2, 3, 4]
        m, n = int(rng.integers(1, 9)), 1
        n = int(rng.integers(1, m + 1))
        tab = {}
        tu1 = int(rng.integers(20_000, 80_000))
        tab[(1, m, 0, 0)] = (tu1, 0)
        tab[(1, 0, n, 0)] = (int(rng.integers(30_000, 90_000)), int(rng.integers(30_000, 90_000)))
        for c in cs:
            tau = int(c * tu1 * rng.uniform(0.98, 1.2))
            tab[(c, m, n, 0)] = (tau, int(tau * rng.uniform(0.3, 1.0)))
        if trial % 5 == 0:                 # exact tie between c = 1 and c = 2 → the smaller c
            tau1, d1 = tab[(1, m, n, 0)]
            tab[(2, m, n, 0)] = (2 * tau1, d1)   # (2τ − 2tu1)/(2tu1) = (τ − tu1)/tu1; same δ
        cmax, cstar, cost = profiler.chunk_choice(tab, cs, m=m, n=n)
        tv0 = tab[(1, 0, n, 0)][1]
        L = {c: sched.chunk_cost(F(1, 2), tab[(c, m, n, 0)][0], tab[(c, m, n, 0)][1], c * tu1, tv0) for c in cs}
        assert cstar == sched.select_c(L), trial
        assert cmax == sched.find_c_max({c: F(tab[(c, m, n, 0)][0], c) for c in cs}, tu1), trial
        for c in cs:
            assert cost[c] == pytest.approx(float(L[c]), rel=1e-12, abs=1e-15)


def test_find_b_max_bitexact_vs_oracle():
    """sd_find_b_max equals oracle.sched.find_b_max on random sub-linear profiles."""
    from fractions import Fraction
    from paper_2605_08835_b200 import profiler
    rng = np.random.default_rng(9)
    for trial in range(300):
        mm = int(rng.integers(2, 17))
        h, a = int(rng.integers(0, 60_000)), int(rng.integers(1_000, 20_000))
        tau = {m: h + a * m + int(rng.integers(0, 3_000)) for m in range(1, mm + 1)}
        tab = {(1, m, 0, 0): (t, 0) for m, t in tau.items()}
        for eps in ((1, 20), (1, 10), (3, 100)):
            assert profiler.find_b_max(tab, mm, eps) == sched.find_b_max(tau, Fraction(*eps)), (trial, eps)

"""Pins for oracle/sched.py and oracle/controller.py (§III-C/§III-D; SPEC.md worked examples).

Golden values with citations: tests/golden/spec_examples.json."""
import json
import os
import time
from fractions import Fraction

import numpy as np
import pytest

from oracle import controller, sched

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_eq2_spec_examples():
    for ex in GOLD["cumulative_latencies"]:
        assert sched.cumulative_latencies(ex["t_u"], ex["t_v"]) == tuple(ex["expect"])


def test_eq2_unet_dominated_identity(rng):
    for _ in range(50):
        c = int(rng.integers(1, 8))
        tv = [int(x) for x in rng.integers(1, 50, c)]
        tu = [v + int(d) for v, d in zip(tv, rng.integers(0, 30, c))]
        Tu, Tv = sched.cumulative_latencies(tu, tv)
        assert Tu == sum(tu) and Tv == Tu - tu[-1] + tv[-1]


def test_eq1_spec_examples():
    for ex in GOLD["chunk_cost"]:
        assert sched.chunk_cost(*ex["args"]) == pytest.approx(ex["expect"], abs=1e-15)
    with pytest.raises(ValueError):
        sched.chunk_cost(0.5, 1, 1, 0, 1)


def test_t_lim():
    assert sched.t_lim(100) == 110 and sched.t_lim(105) == 115 and sched.t_lim(0) == 0
    assert sched.t_lim(100, 0, 10) == 100


def test_validate_spec_examples():
    for ex in GOLD["validate_plan"]:
        bad = sched.validate([tuple(s) for s in ex["plan"]], *ex["window"])
        assert (len(bad) == 0) == ex["ok"], (ex, bad)
        if not ex["ok"]:
            assert ex["violation"] in bad


def random_table(rng, B=6, noise=8):
    """App. B setup: τ ≈ 5 + 20(m − 0.5k)^0.8 + 15n + U{0..8}, δ = τ·U(0.4, 1.0) (int µs·1000)."""
    tab = {}
    for m in range(0, B + 1):
        for n in range(0, B + 1):
            for k in range(0, m + 1):
                if m == 0 and n == 0:
                    continue
                tau = 5 + 20 * max(m - 0.5 * k, 0) ** 0.8 + 15 * n + int(rng.integers(0, noise + 1))
                tau = int(round(tau * 1000))
                delta = int(round(tau * rng.uniform(0.4, 1.0))) if n > 0 else 0
                tab[(m, n, k)] = (tau, delta)
    return tab


def test_exact_dp_equals_bruteforce(rng):
    """I8: the exact (Pareto) DP equals brute force over all ordered stage sequences."""
    n = 0
    for trial in range(12):
        tab = random_table(rng, B=5)
        for M in range(1, 5):
            for N in range(0, 5):
                for K in range(0, M + 1):
                    for a_num in (1, 100):
                        lim = sched.t_lim(sched.tau_ref(tab, M, N, K), a_num, 10) if N else 0
                        if N == 0:
                            continue
                        bf = sched.brute_force(tab, M, N, K, lim)
                        ex = sched.solve_exact(tab, M, N, K, lim)
                        assert bf is not None and ex == bf, (M, N, K, bf, ex)
                        assert sched.validate_with_table(tab, ex[2], M, N, K, lim) == []
                        assert sched.plan_cost(tab, ex[2]) == (ex[0], ex[1])
                        n += 1
    assert n > 500


def test_alg1_is_not_exact_but_feasible(rng):
    """R10: Alg. 1 verbatim is feasible and never better than the optimum; it is sometimes worse."""
    worse = 0
    for trial in range(40):
        tab = random_table(rng, B=5)
        for M in range(2, 6):
            for N in range(1, M + 1):
                for K in range(0, M + 1):
                    lim = sched.t_lim(sched.tau_ref(tab, M, N, K))
                    a1 = sched.solve_alg1(tab, M, N, K, lim)
                    ex = sched.solve_exact(tab, M, N, K, lim)
                    assert a1 is not None and sched.validate_with_table(tab, a1[2], M, N, K, lim) == []
                    assert a1[0] >= ex[0]
                    worse += a1[0] > ex[0]
    assert worse > 0


def test_monotone_in_tlim(rng):
    tab = random_table(rng, B=5)
    for M, N, K in [(4, 3, 2), (5, 5, 1), (3, 4, 0)]:
        base = sched.tau_ref(tab, M, N, K)
        costs = [sched.solve_exact(tab, M, N, K, sched.t_lim(base, a, 10))[0] for a in (0, 1, 3, 10, 100)]
        assert all(costs[i] >= costs[i + 1] for i in range(len(costs) - 1))


def test_spec_single_stage_and_fine_grained():
    """SPEC solve_3ddp examples: M=N=1 → [(1,1,0)]; unconstrained α on a Table-1-shaped table
    prefers the fully fine-grained sequence (Table 1 'VAE latency' ordering)."""
    tab = {(1, 1, 0): (50_000, 30_000), (1, 0, 0): (40_000, 0)}
    assert sched.plan_window(tab, 1, 1, 0) == ((1, 1, 0),)
    # per-pair τ = 46.3 ms, δ = 20.8 ms (SPEC latency.load_table example row); concurrent decodes
    # contend (δ grows as n²), so with unconstrained α the fine-grained plan wins
    t6 = {}
    for m in range(1, 7):
        for n in range(0, m + 1):
            t6[(m, n, 0)] = (46_300 * m, 20_800 * n * n)
    plan = sched.plan_window(t6, 6, 6, 0, a_num=1000, a_den=1)
    assert plan == ((1, 1, 0),) * 6


def test_dp_speed():
    rng = np.random.default_rng(5)
    tab = random_table(rng, B=8)
    t0 = time.perf_counter()
    sched.solve_exact(tab, 8, 8, 8, sched.t_lim(sched.tau_ref(tab, 8, 8, 8)))
    assert time.perf_counter() - t0 < 5.0      # pure Python; the C++ twin is timed separately


def test_map_tasks():
    stages = [(2, 1, 1), (1, 1, 0)]
    unet_tasks = [(10, 5, 20, False), (11, 15, 20, True), (12, 12, 20, True)]
    dec = [(7, 300), (3, 100)]
    m = sched.map_tasks(stages, unet_tasks, dec)
    assert m[0][1] == [11] and m[0][2] == [3] and m[1][2] == [7]
    assert sorted(m[0][0] + m[1][0]) == [10, 11, 12]


def test_p99():
    assert sched.p99(list(range(1, 101))) == 99
    assert sched.p99([5]) == 5


# ---- controller (R15) ----

def _run(ctrl, qs, dt=100_000):
    traj = []
    for i, q in enumerate(qs):
        lv, c, ch = ctrl.decide(i * dt, q)
        traj.append((lv, c))
    return traj


def test_controller_palindrome_and_single_change():
    ctrl = controller.Controller(c_star=1, c_max=3, window=4, h=2)
    rise = [i * 2 for i in range(40)]
    fall = [80 - i * 2 for i in range(40)] + [0] * 60
    traj = _run(ctrl, rise + fall)
    for a, b in zip(traj, traj[1:]):
        assert abs(a[0] - b[0]) + abs(a[1] - b[1]) <= 1
    settings = [traj[0]]
    for s in traj[1:]:
        if s != settings[-1]:
            settings.append(s)
    assert settings == settings[::-1] and max(s[0] for s in settings) == 2 and max(s[1] for s in settings) == 3
    assert traj[-1] == (0, 1)


def test_controller_quiescence():
    ctrl = controller.Controller(c_star=2, c_max=4)
    traj = _run(ctrl, [3, 2, 3, 3, 2, 3] * 10)
    assert all(t == (0, 2) for t in traj)


def test_s_min():
    assert controller.s_min(Fraction(7, 10), 35) == 25 and controller.s_min(Fraction(1, 2), 21) == 11
    assert controller.s_min(None, 30) == 31


ALG1 = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "alg1_trace.json")))


def _alg1_table():
    return {tuple(e["mnk"]): (e["tau"], e["delta"]) for e in ALG1["table"]}


def test_alg1_hand_trace():
    """Alg. 1 against a run traced by hand (tests/golden/alg1_trace.json): every
    successful relaxation in visit order, the strict '<' on line 9, the smallest-u backtrack tie on
    line 16, and the result — which differs from the exact DP's by that tie (R10)."""
    tab, w = _alg1_table(), ALG1["window"]
    lim = sched.t_lim(sched.tau_ref(tab, w["M"], w["N"], w["K"]))
    assert lim == w["T_lim"]
    trace = []
    got = sched.solve_alg1(tab, w["M"], w["N"], w["K"], lim, trace=trace)
    want = [(tuple(r["to"]), r["cost"], r["time"], tuple(r["from"]), tuple(r["action"])) for r in ALG1["relaxations"]]
    assert trace == want
    r = ALG1["alg1_result"]
    assert got == (r["cost"], r["time"], tuple(tuple(s) for s in r["stages"]))
    e = ALG1["exact_result"]
    assert sched.solve_exact(tab, w["M"], w["N"], w["K"], lim) == (e["cost"], e["time"],
                                                                    tuple(tuple(s) for s in e["stages"]))
    assert sched.plan_window(tab, w["M"], w["N"], w["K"], mode="alg1") == tuple(tuple(s) for s in r["stages"])


def test_find_b_max_closed_forms():
    """B_max rule pinned by closed forms: with τ(m) = h + a·m the throughput
    ratio is (m+1)(h + a·m) / (m(h + a·m + a)); the first m where it drops below 1 + ε is found by hand for
    h = 40, a = 10, ε = 1/20: m = 2 gives 3·60/(2·70) = 9/7 > 1.05, …, m = 6: 7·100/(6·110) = 70/66 =
    1.0606 > 1.05, m = 7: 8·110/(7·120) = 88/84 = 1.0476 < 1.05 → B_max = 7. A linear τ = a·m (no fixed cost)
    saturates immediately (ratio 1) → 1; a constant τ has ratio (m+1)/m, which first drops below 1.05 at
    m = 21 (22/21; 21/20 = 1.05 is not below) → 21, or the scan ceiling when that is smaller."""
    aff = {m: 40 + 10 * m for m in range(1, 17)}
    assert sched.find_b_max(aff) == 7
    assert sched.find_b_max({m: 7 * m for m in range(1, 9)}) == 1
    assert sched.find_b_max({m: 100 for m in range(1, 13)}) == 12
    assert sched.find_b_max({m: 100 for m in range(1, 31)}) == 21      # 21/20 = 1.05 is not < 1.05

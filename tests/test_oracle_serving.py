"""Pins for oracle/serving.py (the continuous-batching semantics of SURVEY.md §8(c) steps 1-5).

No paper value fixes a timeline on B200, so the simulator is pinned by closed forms on tables whose
entries are chosen by hand, and by invariants any correct serving loop must satisfy:
  * a lone request: U = n·τ¹(1,0,0), V = U + δ^c(0,1,0) (PAPER.md:289 U_i / V_i; Eq. 2 early release);
  * lockstep requests share rounds (step-level batching);
  * B_max refill happens only at window boundaries, FCFS by (A_i, id) (R16);
  * time-shift invariance of an isolated request; every request takes exactly n_r steps;
  * Skip-CFG only at s_r ≥ s_min_r and only in windows with N > 0 (R6, R8).
"""
import itertools

from oracle import controller as ctl
from oracle import sched, serving


def table(B=8, c_values=(1, 2, 3, 4)):
    """τ^c(m,n,k) = 1000·(2m−k) + 700·n + 50(c−1)·n µs; δ^c(m,n,k) = 600·n + 200·m + 10·k (n > 0)."""
    tabs = {}
    for c in c_values:
        t = {}
        for m, n in itertools.product(range(B + 1), range(B + 1)):
            for k in range(m + 1):
                if m == 0 and n == 0:
                    continue
                tau = 1000 * (2 * m - k) + 700 * n + 50 * (c - 1) * n
                delta = 600 * n + 200 * m + 10 * k if n else 0
                t[(m, n, k)] = (tau, delta)
        tabs[c] = t
    return tabs


def test_lone_request_closed_form():
    tabs = table()
    for n in (1, 3, 20):
        done = serving.simulate([(0, 0, n)], tabs)
        t = done[0]
        assert t.U == n * tabs[1][(1, 0, 0)][0]
        assert t.V == t.U + tabs[1][(0, 1, 0)][1]
        assert t.s == n and t.skips == []


def test_time_shift_invariance():
    tabs = table()
    a = serving.simulate([(5, 0, 7)], tabs)[5]
    b = serving.simulate([(5, 123_456, 7)], tabs)[5]
    assert (b.U - b.A, b.V - b.A) == (a.U - a.A, a.V - a.A)


def test_lockstep_requests_share_rounds():
    tabs = table()
    done = serving.simulate([(i, 0, 4) for i in range(3)], tabs)
    tau3 = tabs[1][(3, 0, 0)][0]
    assert all(done[i].U == 4 * tau3 for i in range(3))
    # the three decodes start at U; whatever plan the DP picks, each ends at a stage start + δ ≥ U + δ(0,1,0)
    assert all(done[i].V >= done[i].U + tabs[1][(0, 1, 0)][1] for i in range(3))


def test_bmax_refill_fcfs():
    """B_max = 2, three requests at t = 0 with one step each: ids 0 and 1 run the first round
    together; id 2 is admitted at the next window boundary (FCFS by (A, id))."""
    tabs = table(B=2, c_values=(1,))
    log = []
    done = serving.simulate([(2, 0, 1), (1, 0, 1), (0, 0, 1)], tabs, b_max=2, c_max=1, log=log)
    tau2 = tabs[1][(2, 0, 0)][0]
    assert done[0].U == done[1].U == tau2
    assert log[0]["M"] == 2 and log[0]["N"] == 0
    assert log[1]["now"] == tau2 and log[1]["M"] == 1 and log[1]["N"] == 2
    assert done[2].U > tau2
    assert all(w["M"] <= 2 and w["N"] <= 2 for w in log)


def test_poisson_invariants():
    tabs = table()
    import random
    rng = random.Random(3)
    trace, t = [], 0
    for i in range(60):
        t += int(rng.expovariate(1 / 4000))
        trace.append((i, t, rng.randint(20, 50)))
    log = []
    done = serving.simulate(trace, tabs, c_star=1, c_max=4, log=log)
    assert sorted(done) == list(range(60))
    for i, a, n in trace:
        d = done[i]
        assert d.A == a and d.s == n
        assert a < d.U < d.V
        assert d.U - a >= n * min(v[0] for v in tabs[1].values() if v[0] > 0) // 8
        lv = [f for f in ctl.LEVELS if f is not None]
        # a skipped step index is at least the loosest possible s_min
        assert all(s >= ctl.s_min(min(lv), n) for s in d.skips)
        assert len(set(d.skips)) == len(d.skips)
    assert all(w["M"] <= 8 and w["K"] <= w["M"] for w in log)
    # the overloaded trace makes the controller escalate at least once, and skips appear
    assert any(w["level"] > 0 for w in log)
    assert sum(len(d.skips) for d in done.values()) > 0


def test_no_skip_without_decodes():
    """R8: windows with N = 0 run (M, 0, 0); a request that never shares a window with a decode is
    never skipped even under an escalated controller."""
    tabs = table()
    done = serving.simulate([(0, 0, 30)], tabs, ctl_kw=dict(up=(-1000, 1)))  # escalate on any slope
    assert done[0].skips == []


def test_metrics_definition():
    tabs = table()
    done = serving.simulate([(0, 0, 2), (1, 10_000, 2)], tabs)
    m = serving.metrics(done)
    e2e = sorted(d.V - d.A for d in done.values())
    assert m["n"] == 2
    assert m["mean_e2e_us"] == sum(e2e) / 2
    assert m["p99_e2e_us"] == e2e[-1]            # ceil(0.99·2) = 2nd smallest
    span = max(d.V for d in done.values()) - 0
    assert abs(m["throughput_per_s"] - 2 / (span / 1e6)) < 1e-12
    assert sched.p99(list(range(1, 101))) == 99


# ---- baseline policies and ablations -------------------------------
def test_serial_closed_form():
    """Diffusers BS = 1: request j starts when request j−1's decode round ends."""
    tabs = table()
    tu, (td_tau, td_delta) = tabs[1][(1, 0, 0)][0], tabs[1][(0, 1, 0)]
    done = serving.simulate([(0, 0, 3), (1, 0, 5), (2, 10**9, 2)], tabs, policy="serial")
    assert done[0].U == 3 * tu and done[0].V == done[0].U + td_delta
    assert done[1].U == done[0].U + td_tau + 5 * tu and done[1].V == done[1].U + td_delta
    assert done[2].U == 10**9 + 2 * tu                        # idle server: starts at its arrival
    assert all(t.skips == [] for t in done.values())


def test_dynamic_batching_closed_form():
    """Dynamic Batching: 0.5 s collection after the oldest request, lockstep until every
    member is done (finished members wait: the straggler effect), synchronous release."""
    tabs = table()
    W = 500_000
    done = serving.simulate([(0, 0, 3), (1, 100_000, 5), (2, 700_000, 2)], tabs, policy="dynamic",
                            dyn_window_us=W)
    t2, t1 = tabs[1][(2, 0, 0)][0], tabs[1][(1, 0, 0)][0]
    assert done[0].U == W + 3 * t2                             # both step together for 3 rounds
    assert done[1].U == done[0].U + 2 * t1                     # the straggler runs on alone
    rel = done[1].U + tabs[1][(0, 2, 0)][0]                    # one decode stage for both
    assert done[0].V == done[1].V == rel                       # all-in-all-out release
    # request 2 arrived during the first batch; its window closes 0.5 s after its arrival
    assert done[2].U == max(rel, 700_000 + W) + 2 * t1
    # a full batch (B_max arrivals) dispatches at the B_max-th arrival, without waiting W
    done = serving.simulate([(i, 1000 * i, 2) for i in range(4)], tabs, b_max=4, policy="dynamic")
    assert done[0].U == 3000 + 2 * tabs[1][(4, 0, 0)][0]


def test_naive_concurrency_runs_full_batch_with_decodes():
    """InstGenIE: every window is one stage (M, min(N, M), 0) at c = 1, never a skip."""
    tabs = table()
    log = []
    trace = [(i, 300_000 * i, 20 + (7 * i) % 13) for i in range(30)]
    done = serving.simulate(trace, tabs, policy="naive", c_star=2, log=log)
    assert len(done) == 30 and all(t.skips == [] for t in done.values())
    for w in log:
        assert w["c"] == 1 and w["level"] == 0
        assert w["stages"] == (((w["M"], min(w["N"], w["M"]), 0),) if w["N"] and w["M"] else
                               ((0, w["N"], 0),) if w["N"] else ((w["M"], 0, 0),))


def test_ablations_disable_their_component():
    tabs = table()
    trace = [(i, 40_000 * i, 20 + (5 * i) % 31) for i in range(60)]          # overload: queue grows
    full = serving.simulate(trace, tabs, c_star=1, c_max=4, ctl_kw=dict(up=(-1000, 1)))
    assert sum(len(t.skips) for t in full.values()) > 0                      # the method skips
    log = []
    no_skip = serving.simulate(trace, tabs, c_star=1, c_max=4, ctl_kw=dict(up=(-1000, 1)), no_skip=True, log=log)
    assert sum(len(t.skips) for t in no_skip.values()) == 0
    assert any(w["c"] > 1 for w in log)                                      # the controller still chunks
    log = []
    no_ctl = serving.simulate(trace, tabs, c_star=1, c_max=4, ctl_kw=dict(up=(-1000, 1)), no_ctl=True, log=log)
    assert all(w["c"] == 1 and w["level"] == 0 for w in log)                 # frozen at its initial state
    for d in (full, no_skip, no_ctl):
        assert len(d) == 60 and all(t.s == t.n and t.A <= t.U <= t.V for t in d.values())


def test_policies_complete_every_request_fcfs_invariants():
    tabs = table()
    trace = [(i, 150_000 * i + (i % 3) * 7, 20 + (11 * i) % 31) for i in range(40)]
    for pol in ("synerdiff", "naive", "dynamic", "serial"):
        done = serving.simulate(trace, tabs, policy=pol)
        assert sorted(done) == list(range(40))
        assert all(t.s == t.n and t.A <= t.U <= t.V for t in done.values()), pol
        if pol == "serial":  # FCFS, one at a time: completions in arrival order, no overlap
            order = sorted(done.values(), key=lambda t: (t.A, t.id))
            assert all(a.V <= b.U for a, b in zip(order, order[1:]))


# ---- mixed resolutions ----------------------------------------------------
def test_mixed_resolution_window_uses_largest_table():
    """A window plans and times with the table of its largest resolution (SPEC S:152 max multiplier):
    a lone small request runs at the small table's τ; once a large request shares its windows, every
    round runs at the large table's τ; a single-resolution trace reproduces the plain simulation."""
    small, big = table(), {c: {k: (3 * v[0], 3 * v[1]) for k, v in t.items()} for c, t in table().items()}
    res = {8: small, 16: big}
    done = serving.simulate([(0, 0, 4, 8)], None, res_tables=res)
    assert done[0].U == 4 * small[1][(1, 0, 0)][0]
    done = serving.simulate([(0, 0, 4, 8), (1, 0, 4, 16)], None, res_tables=res)
    assert done[0].U == done[1].U == 4 * big[1][(2, 0, 0)][0]
    tr = [(i, 200_000 * i, 20 + (7 * i) % 13) for i in range(20)]
    a = serving.simulate(tr, small)
    b = serving.simulate([(i, A, n, 8) for i, A, n in tr], None, res_tables=res)
    assert all((a[i].U, a[i].V) == (b[i].U, b[i].V) for i in a)

"""Offline-profiler formulas and the threshold-aware planner (ORACLE — test infrastructure only).

PAPER.md §III-C (lines 247-262): Eq. 1 chunk cost L(c), Eq. 2 cumulative round latencies,
the C_max 5 % rule. §III-D (lines 284-307): Problem P (Eq. 3a-3f) and Alg. 1 (lines 327-349).

Readings:
  R10  Alg. 1 is not exact for P; `solve_exact` keeps Pareto (cost, time) labels per state;
       `solve_alg1` is Alg. 1 verbatim. Canonical tie-break: (cost, total time, #stages,
       lexicographic (m,n,k) sequence). Actions obey Eq. 3d (1 ≤ m, n ≤ m, k ≤ m).
  R11  τ/δ are integer µs; T_lim = ⌊τ(M,N,K)·(1+α)⌋ with α = α_num/α_den.
  R12  stages are 1…T, τ_0 = 0.
  R13  decode-only stages (m = 0, n ≥ 1, k = 0) are allowed only when N > M; then the reference
       plan for T_lim is [(M, M, K), (0, N−M, 0)] (or [(0, N, 0)] if M = 0).
  R14  mapping E: decodes by (A_i, id); skip slots to eligible tasks with the largest s_r/n_r,
       then id; remaining UNet slots in batch order.
A table is a dict {(m, n, k): (tau_us, delta_us)} for the current chunk granularity c.
"""
from __future__ import annotations

from fractions import Fraction
from itertools import product


# ---- Eq. 1 / Eq. 2 ---------------------------------------------------------------------------

def cumulative_latencies(t_u, t_v):
    """Eq. 2: T_u(c) = Σ_{i≤c} max(t_u^i, t_v^i);  T_v(c) = Σ_{i<c} max(t_u^i, t_v^i) + t_v^c."""
    assert len(t_u) == len(t_v) and len(t_u) >= 1
    c = len(t_u)
    Tu = sum(max(a, b) for a, b in zip(t_u, t_v))
    Tv = sum(max(t_u[i], t_v[i]) for i in range(c - 1)) + t_v[c - 1]
    return Tu, Tv


def chunk_cost(lam, Tu, Tv, Tu0, Tv0):
    """Eq. 1: L(c) = λ·(T_u(c)−T_u0)/T_u0 + (1−λ)·(T_v(c)−T_v0)/T_v0."""
    if Tu0 <= 0 or Tv0 <= 0:
        raise ValueError("zero baseline")
    return lam * (Tu - Tu0) / Tu0 + (1 - lam) * (Tv - Tv0) / Tv0


def select_c(costs_by_c):
    """c* = argmin_c L(c), ties to the smaller c (R31). costs_by_c: {c: L(c)}."""
    return min(sorted(costs_by_c), key=lambda c: (costs_by_c[c], c))


def find_b_max(tau_solo_us_by_m, eps=Fraction(1, 20)):
    """Saturation batch B_max ("the saturation batch size B_max based on the sub-linear
    scaling of throughput"; SPEC find_b_max S:202-210): throughput(m) = m / τ(m, 0, 0); B_max = the
    smallest m with throughput(m+1)/throughput(m) − 1 < ε; the largest profiled m if none (never
    saturates). Exact in Fractions. tau_solo_us_by_m: {m: τ(m, 0, 0) µs} for m = 1 … m_max."""
    ms = sorted(tau_solo_us_by_m)
    assert ms == list(range(1, len(ms) + 1)), "profile m = 1 .. m_max"
    thr = {m: Fraction(m, tau_solo_us_by_m[m]) for m in ms}
    for m in ms[:-1]:
        if thr[m + 1] / thr[m] - 1 < eps:
            return m
    return ms[-1]


def find_c_max(concurrent_unet_us_by_c, solo_unet_us, num=5, den=100):
    """C_max = largest c whose concurrent UNet round ≤ (1 + 5 %)·solo; ≥ 1."""
    ok = [c for c, t in concurrent_unet_us_by_c.items() if t * den <= solo_unet_us * (den + num)]
    return max(ok) if ok else 1


# ---- Problem P --------------------------------------------------------------------------------

def t_lim(tau_ref_us: int, a_num: int = 1, a_den: int = 10) -> int:
    """R11: ⌊τ·(1+α)⌋ = (τ·α_den + τ·α_num) // α_den."""
    return (tau_ref_us * a_den + tau_ref_us * a_num) // a_den


def reference_plan(M, N, K):
    if N <= M:
        return [(M, N, K)]
    if M == 0:
        return [(0, N, 0)]
    return [(M, M, K), (0, N - M, 0)]


def tau_ref(table, M, N, K):
    return sum(table[s][0] for s in reference_plan(M, N, K))


def actions(i, j, u, M, N, K):
    """Valid actions from state (i, j, u) in canonical (lexicographic) order (Eq. 3d, R13)."""
    out = []
    decode_only = N > M
    for m, n, k in product(range(0, M - i + 1), range(0, N - j + 1), range(0, K - u + 1)):
        if m >= 1:
            if n <= m and k <= m:
                out.append((m, n, k))
        elif decode_only and n >= 1 and k == 0:
            out.append((m, n, k))
    return out


def plan_cost(table, stages):
    """Σ_t n_t·V(t) with V(t) = Σ_{j<t} τ_j + δ_t (Eq. 3a/3b minus the constant Σ(U_i − A_i));
    returns (cost, total time)."""
    time = cost = 0
    for (m, n, k) in stages:
        tau, delta = table[(m, n, k)]
        if n > 0:
            cost += n * (time + delta)
        time += tau
    return cost, time


def validate(stages, M, N, K):
    """Eq. 3c-3e (+ R13). Returns the list of violated constraint names."""
    bad = []
    if sum(s[0] for s in stages) != M:
        bad.append("sum m_t = M")
    if sum(s[1] for s in stages) != N:
        bad.append("sum n_t = N")
    for m, n, k in stages:
        if m >= 1 and not (0 <= n <= m):
            bad.append("n_t <= m_t")
        if not (0 <= k <= m):
            bad.append("k_t <= m_t")
        if m == 0 and not (N > M and n >= 1 and k == 0):
            bad.append("decode-only stage")
    if sum(s[2] for s in stages) > K:
        bad.append("sum k_t <= K")
    return bad


def validate_with_table(table, stages, M, N, K, limit):
    """Eq. 3c-3f."""
    bad = validate(stages, M, N, K)
    if sum(table[s][0] for s in stages) > limit:
        bad.append("sum tau <= (1+alpha) tau(M,N,K)")
    return bad


def _key(label):
    cost, time, seq = label
    return (cost, time, len(seq), seq)


def brute_force(table, M, N, K, limit):
    """Enumerate every ordered stage sequence satisfying Eq. 3c-3f; best by the canonical key."""
    best = None

    def rec(i, j, u, time, cost, seq):
        nonlocal best
        if i == M and j == N:
            lab = (cost, time, tuple(seq))
            if best is None or _key(lab) < _key(best):
                best = lab
            # an empty continuation is the only one: all further actions need m ≥ 1 or n ≥ 1
            return
        for a in actions(i, j, u, M, N, K):
            tau, delta = table[a]
            tn = time + tau
            if tn > limit:
                continue
            cn = cost + (a[1] * (time + delta) if a[1] > 0 else 0)
            seq.append(a)
            rec(i + a[0], j + a[1], u + a[2], tn, cn, seq)
            seq.pop()

    rec(0, 0, 0, 0, 0, [])
    return best          # (cost, time, stages) or None if infeasible


def solve_exact(table, M, N, K, limit):
    """Exact DP for P (R10): Pareto labels (cost, time) per state (i, j, u), dominance pruning,
    canonical tie-break among equal (cost, time). Returns (cost, time, stages) or None."""
    labels = {(0, 0, 0): [(0, 0, ())]}
    order = sorted(product(range(M + 1), range(N + 1), range(K + 1)))
    for st in order:
        if st not in labels:
            continue
        i, j, u = st
        for a in actions(i, j, u, M, N, K):
            tau, delta = table[a]
            nxt = (i + a[0], j + a[1], u + a[2])
            for cost, time, seq in labels[st]:
                tn = time + tau
                if tn > limit:
                    continue
                cn = cost + (a[1] * (time + delta) if a[1] > 0 else 0)
                _insert(labels.setdefault(nxt, []), (cn, tn, seq + (a,)))
    finals = [lab for u in range(K + 1) for lab in labels.get((M, N, u), [])]
    if not finals:
        return None
    return min(finals, key=_key)


def _insert(lst, lab):
    c, t, seq = lab
    for idx, (c2, t2, s2) in enumerate(lst):
        if c2 <= c and t2 <= t and (c2 < c or t2 < t):
            return                                   # dominated
        if c2 == c and t2 == t:
            if (len(seq), seq) < (len(s2), s2):
                lst[idx] = lab
            return
    lst[:] = [x for x in lst if not (c <= x[0] and t <= x[1])]
    lst.append(lab)
    lst.sort()


def solve_alg1(table, M, N, K, limit, trace=None):
    """Alg. 1 verbatim: one ⟨cost, time⟩ per state, relax on strictly smaller
    cost; states and actions visited in ascending lexicographic order; backtrack from
    argmin_u DP[M,N,u].c (ties → smallest u). Returns (cost, time, stages) or None."""
    INF = None
    dp = {}
    par = {}
    dp[(0, 0, 0)] = (0, 0)
    for st in sorted(product(range(M + 1), range(N + 1), range(K + 1))):
        if st not in dp:                                  # DP[i,j,u].c = ∞
            continue
        i, j, u = st
        c0, t0 = dp[st]
        for a in actions(i, j, u, M, N, K):
            tau, delta = table[a]
            t_new = t0 + tau
            if t_new <= limit:
                cv = (t0 + delta) if a[1] > 0 else 0
                c_new = c0 + cv * a[1]
                nxt = (i + a[0], j + a[1], u + a[2])
                if nxt not in dp or c_new < dp[nxt][0]:
                    dp[nxt] = (c_new, t_new)
                    par[nxt] = (st, a)
                    if trace is not None:
                        trace.append((nxt, c_new, t_new, st, a))
    ends = [(dp[(M, N, u)][0], u) for u in range(K + 1) if (M, N, u) in dp]
    if not ends:
        return INF
    _, u = min(ends)
    st = (M, N, u)
    seq = []
    while st != (0, 0, 0):
        prev, a = par[st]
        seq.append(a)
        st = prev
    seq.reverse()
    cost, time = plan_cost(table, seq)
    assert cost == dp[(M, N, u)][0]
    return (cost, time, tuple(seq))


def plan_window(table, M, N, K, a_num=1, a_den=10, mode="exact"):
    """§8(c) step 3: N = 0 → one round (M, 0, 0) (R8); else T_lim, solve, fall back to the
    reference plan if nothing is feasible (cannot happen: the reference plan meets T_lim)."""
    if M == 0 and N == 0:
        return ()
    if N == 0:
        return ((M, 0, 0),)
    lim = t_lim(tau_ref(table, M, N, K), a_num, a_den)
    sol = (solve_exact if mode == "exact" else solve_alg1)(table, M, N, K, lim)
    if sol is None:
        return tuple(reference_plan(M, N, K))
    return sol[2]


def map_tasks(stages, unet_tasks, decode_tasks):
    """R14. unet_tasks: [(id, s, n_steps, eligible)] in batch order; decode_tasks: [(id, A)].
    Returns per stage (unet_ids, skip_ids, decode_ids)."""
    dec = sorted(decode_tasks, key=lambda d: (d[1], d[0]))
    elig = sorted([t for t in unet_tasks if t[3]], key=lambda t: (-Fraction(t[1], t[2]), t[0]))
    n_skip = sum(s[2] for s in stages)
    skippers = [t[0] for t in elig[:n_skip]]
    rest = [t[0] for t in unet_tasks if t[0] not in set(skippers)]
    out = []
    di = si = ri = 0
    for m, n, k in stages:
        skip_ids = skippers[si:si + k]
        si += k
        u_ids = list(skip_ids) + rest[ri:ri + (m - k)]
        ri += m - k
        out.append((u_ids, skip_ids, [d[0] for d in dec[di:di + n]]))
        di += n
    return out


def expand_rounds(stages, c):
    """R9: a stage at granularity c is c consecutive rounds of the same (m, n, k); each decode in
    the stage runs chunk ρ in round ρ. Returns [(stage_index, round_in_stage)]."""
    return [(t, r) for t in range(len(stages)) for r in range(c)]


def p99(values):
    """Ceil-rank order statistic (R18; SPEC engine.compute_metrics)."""
    v = sorted(values)
    n = len(v)
    r = -(-99 * n // 100)
    return v[max(r, 1) - 1]

"""Continuous-batching serving semantics on a virtual clock (ORACLE — test infrastructure only).

The plain algorithm of SURVEY.md §8(c) steps 1-5 (PAPER.md:66 step-level scheduling and refill;
:289-307 Problem P, threshold-aware plan, controller; :262 Eq. 2 final-round early release),
with round durations taken from the τ/δ table instead of a GPU (SPEC.md's simulator idea).
The C++ serving loop in virtual-clock mode must reproduce every decision and timestamp bit-exactly.

Per window:
  1. admit arrived requests (A_i ≤ now) FCFS by (A_i, id) until the batch holds B_max (R16);
  2. M = |batch|, decode-pending D sorted by (A_i, id), N = min(|D|, B_max); with the controller's
     level f: s_min_r = ⌈f·n_r⌉, K = #{r : s_r ≥ s_min_r} (R6);
  3. N = 0 → one round (M, 0, 0) from the c = 1 table (R8); else plan (S, E) at the current c
     (R10, R11, R13, R14) and run every stage as c rounds (R9);
  4. a stage (m, n, k) lasts τ^c(m,n,k) split into c rounds (⌊τ/c⌋ each, the remainder in the last);
     each of its UNet tasks takes one step per round (its k skip tasks without the uncond row);
     a task reaching n_r stamps U_r at that round's end and becomes decode-pending; each of the
     stage's decodes completes at stage start + δ^c(m,n,k) (Eq. 2) and stamps V_r;
  5. the controller observes (now, waiting queue) after the window (R15).

Baseline policies and ablations (PAPER.md:316-324 §IV Baselines, :395-397 §IV-E Ablation; SURVEY
§8(f) rank 1), on the same table and clock:
  "serial"   Diffusers, BS = 1: FCFS, one request at a time, every step a (1, 0, 0) round,
             then its whole decode (0, 1, 0); the next request is admitted after the decode.
  "dynamic"  Dynamic Batching: a batch is collected for 0.5 s after its oldest request
             (or until B_max have arrived) — dispatched at max(now, min(A_first + W, A_{B_max-th})) —
             then stepped in lockstep rounds (m_active, 0, 0) until EVERY member is done (all-in-
             all-out: finished members wait, the straggler effect P:40); then the batch is decoded
             in stages (0, ≤ n_max, 0) and released together (every V_i = the release time).
  "naive"    InstGenIE: continuous batching with direct UNet-VAE concurrency — per window one
             stage (M, min(N, M), 0) (or (0, N, 0) with no UNet work), c = 1, no Skip-CFG, no
             threshold plan, no controller.
  ablations  of "synerdiff": no_skip (level pinned to 0: no Skip-CFG), no_ctl (controller frozen at
             its initial state); "no chunking" is c_star = c_max = 1.

Mixed resolutions (PAPER.md:315 mixes 512/768/1024; reading R22 extended by the
build): trace entries may carry a 4th field, the request's latent size r. With `res_tables`
{r: {c: table}}, every window plans and times its stages with the table of the LARGEST resolution
among its batch and its decode-pending requests (SPEC's "max multiplier"); the serial policy
uses each request's own table, dynamic batching the batch's largest. On the GPU a round runs one
sd_step_batch per resolution group of the stepping tasks.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import controller as ctl
from . import sched


@dataclass
class Task:
    id: int
    A: int
    n: int
    r: int = 0          # latent size (mixed-resolution traces); 0 = the single table
    g: float = 7.5
    s: int = 0
    U: int | None = None
    V: int | None = None
    skips: list = field(default_factory=list)


def _tasks(trace):
    return sorted((Task(e[0], e[1], e[2], e[3] if len(e) > 3 else 0) for e in trace), key=lambda t: (t.A, t.id))


def simulate(trace, tables, b_max=8, a_num=1, a_den=10, mode="exact", c_star=1, c_max=4, ctl_kw=None,
             log=None, policy="synerdiff", no_skip=False, no_ctl=False, dyn_window_us=500_000, n_max=None,
             res_tables=None):
    """trace: [(id, arrival_us, n_steps[, latent_r])], tables: {c: {(m,n,k): (tau_us, delta_us)}};
    res_tables (mixed resolutions): {r: {c: {...}}} — then `tables` is unused.
    Returns {id: Task}. `log` (list) receives one dict per window."""
    n_max = b_max if n_max is None else n_max
    pick = (lambda ts: res_tables[max(t.r for t in ts)]) if res_tables else (lambda ts: tables)
    if policy == "serial":
        return _serial(trace, pick)
    if policy == "dynamic":
        return _dynamic(trace, pick, b_max, n_max, dyn_window_us)
    srv = Server(trace, pick, b_max, a_num, a_den, mode, c_star, c_max, ctl_kw, log, policy, no_skip, no_ctl, n_max)
    while srv.window() != "done":
        pass
    return srv.done


class Server:
    """The SynerDiff / naive loop of `simulate` as a stepping object, so several of them (one per rank,
    SURVEY §8(e)) can run in lockstep with the C1 all-gather between windows. window() runs one
    window ("ran"), or, with nothing admitted, jumps the clock to the next arrival ("idle"), or reports
    "done". With a global snapshot set (set_global_load, P > 1) the controller observes the summed
    waiting queue of the snapshot instead of this server's own (R15; the GPU server's rule)."""

    def __init__(self, trace, pick, b_max, a_num, a_den, mode, c_star, c_max, ctl_kw, log, policy, no_skip, no_ctl,
                 n_max):
        self.pick, self.b_max, self.a_num, self.a_den, self.mode = pick, b_max, a_num, a_den, mode
        self.log, self.naive, self.no_skip, self.no_ctl, self.n_max = log, policy == "naive", no_skip, no_ctl, n_max
        self.pending = _tasks(trace)
        self.pi = 0
        self.batch, self.dec, self.done = [], [], {}
        self.now = 0
        self.C = ctl.Controller(c_star=c_star, c_max=c_max, **(ctl_kw or {}))
        self.global_load = None

    def set_global_load(self, loads):
        """loads: [P][4] ints (waiting, decode-pending, active, completed) — the C1 snapshot."""
        self.global_load = [list(r) for r in loads]

    def load(self):
        waiting = sum(1 for t in self.pending[self.pi:] if t.A <= self.now)
        return [waiting, len(self.dec), len(self.batch), len(self.done)]

    def window(self):
        if not (self.pi < len(self.pending) or self.batch or self.dec):
            return "done"
        pending, b_max, naive = self.pending, self.b_max, self.naive
        batch, dec = self.batch, self.dec
        while self.pi < len(pending) and pending[self.pi].A <= self.now and len(batch) < b_max:
            batch.append(pending[self.pi])
            self.pi += 1
        if not batch and not dec:
            self.now = pending[self.pi].A
            return "idle"
        level, c = self.C.level, self.C.c
        if self.no_skip or naive:
            level = 0
        if naive:
            c = 1
        f = ctl.LEVELS[level]
        M = len(batch)
        dq = sorted(dec, key=lambda t: (t.A, t.id))[:min(b_max, self.n_max)]
        N = len(dq)
        tabs_w = self.pick(batch + dq)   # mixed resolutions: the table of the window's largest resolution
        elig = [t.s >= ctl.s_min(f, t.n) for t in batch]
        K = sum(elig)
        if N == 0:
            stages, tc, rounds = ((M, 0, 0),), 1, 1
        elif naive:
            stages, tc, rounds = (((M, min(N, M), 0),) if M else ((0, N, 0),)), 1, 1
        else:
            stages = sched.plan_window(tabs_w[c], M, N, K, self.a_num, self.a_den, self.mode)
            tc, rounds = c, c
        tab = tabs_w[tc]
        mapping = sched.map_tasks(stages, [(t.id, t.s, t.n, e) for t, e in zip(batch, elig)],
                                  [(t.id, t.A) for t in dq])
        by_id = {t.id: t for t in batch + dq}
        if self.log is not None:
            self.log.append(dict(now=self.now, M=M, N=N, K=K, level=level, c=c, stages=tuple(stages)))
        for (m, n, k), (u_ids, skip_ids, d_ids) in zip(stages, mapping):
            tau, delta = tab[(m, n, k)]
            t0 = self.now
            per, rem = divmod(tau, rounds)
            for rho in range(rounds):
                self.now += per + (rem if rho == rounds - 1 else 0)
                for uid in u_ids:
                    t = by_id[uid]
                    if t.s >= t.n:
                        continue
                    if uid in skip_ids:
                        t.skips.append(t.s)
                    t.s += 1
                    if t.s == t.n:
                        t.U = self.now
                        batch.remove(t)
                        dec.append(t)
            for did in d_ids:
                t = by_id[did]
                t.V = t0 + delta
                dec.remove(t)
                self.done[t.id] = t
        waiting = sum(1 for t in pending[self.pi:] if t.A <= self.now)
        gw = waiting if not self.global_load or len(self.global_load) <= 1 else sum(r[0] for r in self.global_load)
        if not (naive or self.no_ctl):
            self.C.decide(self.now, gw)
        if self.log is not None:
            self.log[-1].update(end=self.now, waiting=gw, level_after=self.C.level, c_after=self.C.c)
        return "ran"


def simulate_sharded(trace, P, tables, max_epochs=1_000_000, **kw):
    """SURVEY §8(e) on a virtual clock: P servers, each on the shard {id : id mod P = rank} (R32), run in
    lockstep epochs; in each epoch every server runs one window step (Server.window), then the C1
    all-gather hands every server the same [P][4] snapshot of all loads (taken after the epoch).
    Returns ({id: Task} per rank, [per-rank window logs])."""
    pick = lambda ts: tables  # noqa: E731 (one resolution)
    logs = [[] for _ in range(P)]
    args = dict(b_max=8, a_num=1, a_den=10, mode="exact", c_star=1, c_max=4, ctl_kw=None, policy="synerdiff",
                no_skip=False, no_ctl=False, n_max=None)
    args.update(kw)
    args["n_max"] = args["b_max"] if args["n_max"] is None else args["n_max"]
    srv = [Server([e for e in trace if e[0] % P == r], pick, args["b_max"], args["a_num"], args["a_den"],
                  args["mode"], args["c_star"], args["c_max"], args["ctl_kw"], logs[r], args["policy"],
                  args["no_skip"], args["no_ctl"], args["n_max"]) for r in range(P)]
    for _ in range(max_epochs):
        states = [s.window() for s in srv]
        if all(x == "done" for x in states):
            break
        snap = [s.load() for s in srv]
        for s in srv:
            s.set_global_load(snap)
    return [s.done for s in srv], logs


def _serial(trace, pick):
    """Diffusers baseline: BS = 1, FCFS, denoise then decode, one request at a time."""
    done, now = {}, 0
    for t in _tasks(trace):
        tab = pick([t])[1]
        now = max(now, t.A)
        tau, _ = tab[(1, 0, 0)]
        for _ in range(t.n):
            now += tau
            t.s += 1
        t.U = now
        tau, delta = tab[(0, 1, 0)]
        t.V = now + delta
        now += tau
        done[t.id] = t
    return done


def _dynamic(trace, pick, b_max, n_max, window_us):
    """Dynamic Batching baseline: collection window, lockstep, synchronous release."""
    pending = _tasks(trace)
    done, now, pi = {}, 0, 0
    while pi < len(pending):
        first = pending[pi].A
        full = pending[pi + b_max - 1].A if pi + b_max - 1 < len(pending) else None
        close = first + window_us if full is None else min(first + window_us, full)
        now = max(now, close)
        batch = []
        while pi < len(pending) and len(batch) < b_max and pending[pi].A <= now:
            batch.append(pending[pi])
            pi += 1
        tab = pick(batch)[1]
        while any(t.s < t.n for t in batch):
            active = [t for t in batch if t.s < t.n]
            now += tab[(len(active), 0, 0)][0]
            for t in active:
                t.s += 1
                if t.s == t.n:
                    t.U = now
        for j in range(0, len(batch), n_max):
            now += tab[(0, min(n_max, len(batch) - j), 0)][0]
        for t in batch:
            t.V = now
            done[t.id] = t
    return done


def metrics(done):
    """R18: throughput = completed / (last V − first A); mean E2E; P99 by ceil rank."""
    e2e = [t.V - t.A for t in done.values()]
    span = max(t.V for t in done.values()) - min(t.A for t in done.values())
    return dict(n=len(e2e), throughput_per_s=len(e2e) / (span / 1e6) if span > 0 else 0.0,
                mean_e2e_us=sum(e2e) / len(e2e), p99_e2e_us=sched.p99(e2e))

"""Load-adaptive feedback controller (ORACLE — test infrastructure only).

PAPER.md:307 (§III-D): "Upon detecting queue buildup, the controller raises the quality
threshold S to increase Skip-CFG frequency and boost throughput, while restoring it as load
subsides … If throughput remains insufficient even at the minimum quality threshold S_min, the
controller increments VAE Chunking granularity c". No numbers are given; reading R15:
  signal = waiting-queue length (global: summed over ranks from the all-gather);
  least-squares slope over the last W = 10 samples, times in µs;
  θ_up = +1/2 task/s, θ_down = −1/5 task/s, hysteresis h = 3 consecutive decides;
  escalate level first, then c; de-escalate c first, then level; ≤ 1 change per decide.
Levels (R6): f ∈ {∞ (no skip), 0.7, 0.5}; s_min_r = ⌈f·n_r⌉.
All comparisons are exact integer/rational arithmetic.
"""
from __future__ import annotations

from fractions import Fraction

LEVELS = (None, Fraction(7, 10), Fraction(1, 2))


class Controller:
    def __init__(self, c_star=1, c_max=16, window=10, up=(1, 2), down=(-1, 5), h=3, levels=LEVELS):
        self.level = 0
        self.c = c_star
        self.c_star = c_star
        self.c_max = c_max
        self.window = window
        self.up = Fraction(*up) / 1_000_000        # per µs
        self.down = Fraction(*down) / 1_000_000
        self.h = h
        self.levels = levels
        self.samples = []
        self.n_up = 0
        self.n_down = 0

    def observe(self, now_us: int, queue: int):
        if self.samples and now_us < self.samples[-1][0]:
            raise ValueError("time regression")
        self.samples.append((int(now_us), int(queue)))
        if len(self.samples) > self.window:
            self.samples.pop(0)

    def slope(self):
        """Least-squares slope (tasks per µs) as a Fraction, or None if undefined."""
        if len(self.samples) < 2:
            return None
        t0 = self.samples[0][0]
        n = len(self.samples)
        st = sum(t - t0 for t, _ in self.samples)
        sq = sum(q for _, q in self.samples)
        stt = sum((t - t0) ** 2 for t, _ in self.samples)
        stq = sum((t - t0) * q for t, q in self.samples)
        den = n * stt - st * st
        if den == 0:
            return None
        return Fraction(n * stq - st * sq, den)

    def decide(self, now_us: int, queue: int):
        """observe + decide; returns (level, c, changed)."""
        self.observe(now_us, queue)
        s = self.slope()
        changed = False
        if s is None:
            return self.level, self.c, changed
        if s > self.up:
            self.n_up += 1
            self.n_down = 0
        elif s < self.down:
            self.n_down += 1
            self.n_up = 0
        else:
            self.n_up = self.n_down = 0
        if self.n_up >= self.h:
            self.n_up = 0
            if self.level < len(self.levels) - 1:
                self.level += 1
                changed = True
            elif self.c < self.c_max:
                self.c += 1
                changed = True
        elif self.n_down >= self.h:
            self.n_down = 0
            if self.c > self.c_star:
                self.c -= 1
                changed = True
            elif self.level > 0:
                self.level -= 1
                changed = True
        return self.level, self.c, changed


def s_min(level_f, n_steps):
    """R6: s_min = ⌈f·n⌉; f = None → no step is eligible."""
    if level_f is None:
        return n_steps + 1
    return -((-level_f.numerator * n_steps) // level_f.denominator)

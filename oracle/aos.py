"""Adaptive operator selection + profile priors (test infrastructure only).

Restates `aos.py:22-186` and `profiles.py:42-108`.  Python's builtin `sum`
is used wherever the reference uses it: on CPython >= 3.12 it is Neumaier
compensated summation, which the device code replicates (see
`neumaier_sum` below, used only to test that claim).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .moves import BUILTINS, CROSSOVER_IDS, LNS_IDS, OR_OPT, THREE_OPT, applicable

DEFAULT_K = (0.8, 0.15, 0.05)  # aos.py:19


@dataclass(frozen=True)
class AosCfg:
    """aos.py:22-38 defaults."""

    interval: int = 10
    alpha: float = 0.7
    floor: float = 0.01
    cap: float = 0.6
    eps: float = 1e-6
    stagnation: int = 5


class Entry:
    __slots__ = ("id", "name", "fn", "w", "floor", "cap")

    def __init__(self, seq_id, name, fn, w=1.0, floor=0.0, cap=math.inf):
        self.id, self.name, self.fn, self.w, self.floor, self.cap = \
            seq_id, name, fn, w, floor, cap


class Registry:
    """operators.py:91-127."""

    def __init__(self, entries):
        self.entries = list(entries)
        self.normalize()

    def normalize(self):
        total = sum(e.w for e in self.entries)
        for e in self.entries:
            e.w /= total

    def ids(self):
        return [e.id for e in self.entries]

    def weights(self):
        return [e.w for e in self.entries]

    def get(self, seq_id):
        for e in self.entries:
            if e.id == seq_id:
                return e
        raise KeyError(seq_id)


def build_registry(spec, allowed=None) -> Registry:
    """operators.py:618-624; `allowed` restricts the id set (used to compare
    engines on a common operator subset)."""
    return Registry([Entry(i, name, fn) for i, name, fn in BUILTINS
                     if applicable(i, spec) and (allowed is None or i in allowed)])


PRESETS = {  # profiles.py:42-46 (three_opt, or_opt, lns, lns_cap)
    "small": (0.50, 0.80, 0.006, 0.02),
    "medium": (0.30, 0.70, 0.004, 0.01),
    "large": (0.05, 0.30, 0.001, 0.005),
}


def scale_of(spec) -> str:
    """profiles.py:65-73."""
    return "small" if spec.d2 <= 100 else ("medium" if spec.d2 <= 250 else "large")


def apply_preset(reg: Registry, scale: str, p_cross: float = 0.1):
    """profiles.py:76-108."""
    three, oro, lns, lns_cap = PRESETS[scale]
    xs = []
    plain = 0.0
    for e in reg.entries:
        if e.id == THREE_OPT:
            e.w = three
        elif e.id == OR_OPT:
            e.w = oro
        elif e.id in LNS_IDS:
            e.w, e.cap = lns, lns_cap
        elif e.id in CROSSOVER_IDS:
            xs.append(e)
            continue
        else:
            e.w = 1.0
        plain += e.w
    if xs:
        share = p_cross / (1.0 - p_cross) * plain
        for e in xs:
            e.w = share / len(xs)
    reg.normalize()


def add_custom(reg: Registry, seq_id, name, fn, weight):
    """operators.py:666-668 — append then renormalise (per registration)."""
    reg.entries.append(Entry(seq_id, name, fn, w=weight))
    reg.normalize()


def sample_k(kw, rng) -> int:
    """aos.py:147-154."""
    x = rng.random() * (kw[0] + kw[1] + kw[2])
    if x < kw[0]:
        return 1
    if x < kw[0] + kw[1]:
        return 2
    return 3


def sample_seq(reg: Registry, rng) -> int:
    """aos.py:157-175 (no `applicable` filter on the engine path)."""
    total = sum(e.w for e in reg.entries)
    x = rng.random() * total
    acc = 0.0
    for e in reg.entries:
        acc += e.w
        if x < acc:
            return e.id
    return reg.entries[-1].id


def ema(w, u, v, cfg: AosCfg) -> float:
    """aos.py:96-100."""
    return cfg.alpha * w + (1.0 - cfg.alpha) * (v / (u + cfg.eps) + cfg.floor)


def window(seq_floor, seq_cap, cfg: AosCfg):
    """aos.py:103-113."""
    lo = max(cfg.floor, seq_floor)
    hi = min(cfg.cap, seq_cap)
    return (hi if hi < lo else lo), hi


def update_weights(reg: Registry, usage, impr, cfg: AosCfg):
    """aos.py:116-134 (returns the pre-normalisation weights).

    Type fidelity matters here: the reference stores each clamped weight
    into a numpy array and reads it back (aos.py:124-130), so from the first
    update on every sequence weight is an `np.float64`.  CPython's `sum()`
    only applies Neumaier compensation to exact `float` items, hence every
    later `sum(e.weight ...)` (operators.py:114, aos.py:169) is a plain
    left-to-right sum.  The device replicates exactly this: host-provided
    initial totals (compensated), device-updated totals sequential.
    """
    pre = np.empty(len(reg.entries))
    for i, (e, u, v) in enumerate(zip(reg.entries, usage, impr)):
        lo, hi = window(e.floor, e.cap, cfg)
        pre[i] = min(max(ema(e.w, int(u), int(v), cfg), lo), hi)
        e.w = pre[i]
    reg.normalize()
    return pre


def update_k(kw, k_usage, k_impr, cfg: AosCfg):
    """aos.py:137-144."""
    new = [max(ema(w, int(u), int(v), cfg), cfg.floor) for w, u, v in zip(kw, k_usage, k_impr)]
    total = sum(new)
    return tuple(w / total for w in new)


def stagnation(count, kw, cfg: AosCfg):
    """aos.py:178-186."""
    if count > cfg.stagnation:
        return DEFAULT_K, 0
    return tuple(kw), count


def neumaier_sum(values) -> float:
    """The algorithm CPython 3.12's builtin sum() applies to floats (the
    first float joins the integer start 0 exactly), restated so tests can
    show builtin sum == this == the device routine."""
    it = iter(values)
    try:
        s = float(next(it))
    except StopIteration:
        return 0
    c = 0.0
    for x in it:
        t = s + x
        if abs(s) >= abs(x):
            c += (s - t) + x
        else:
            c += (x - t) + s
        s = t
    if c and math.isfinite(c):
        s += c
    return s

"""Operator catalogue and registry — API mirror of the reference's
`operators.py` (ids :29-51, CustomOperator :79-88, SequenceRegistry :91-127,
build_registry :618-624, register_custom :634-669).

The operators themselves run on the device (kernels/go_perm.cuh).  A
`CustomOperator` carries a CUDA snippet (`cuda`), compiled with NVRTC into the
evolve kernel — the paper's JIT injection (§3.3.2); its Python
`apply` is kept only for source compatibility and is never executed.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable

from .core import EncodingKind, ProblemConfig, RowModeKind

SEQ_SWAP, SEQ_INSERT, SEQ_REVERSE, SEQ_OR_OPT, SEQ_THREE_OPT = 0, 1, 2, 3, 4
SEQ_FLIP, SEQ_SEG_FLIP, SEQ_RANDOM_RESET, SEQ_SEG_RESET = 5, 6, 7, 8
SEQ_ROW_SWAP, SEQ_ROW_SPLIT, SEQ_ROW_MERGE = 9, 10, 11
SEQ_OX_CROSSOVER, SEQ_UNIFORM_CROSSOVER = 12, 13
SEQ_SEG_SHUFFLE, SEQ_SCATTER_SHUFFLE, SEQ_GUIDED_REBUILD = 14, 15, 16
CUSTOM_ID_START = 100
RESERVED_BAND = (32, 100)
LNS_IDS = (SEQ_SEG_SHUFFLE, SEQ_SCATTER_SHUFFLE, SEQ_GUIDED_REBUILD)
CROSSOVER_IDS = (SEQ_OX_CROSSOVER, SEQ_UNIFORM_CROSSOVER)

BUILTIN_NAMES = {
    SEQ_SWAP: "swap", SEQ_INSERT: "insert", SEQ_REVERSE: "reverse", SEQ_OR_OPT: "or_opt",
    SEQ_THREE_OPT: "three_opt", SEQ_FLIP: "flip", SEQ_SEG_FLIP: "seg_flip",
    SEQ_RANDOM_RESET: "random_reset", SEQ_SEG_RESET: "seg_reset", SEQ_ROW_SWAP: "row_swap",
    SEQ_ROW_SPLIT: "row_split", SEQ_ROW_MERGE: "row_merge", SEQ_OX_CROSSOVER: "ox_crossover",
    SEQ_UNIFORM_CROSSOVER: "uniform_crossover", SEQ_SEG_SHUFFLE: "seg_shuffle",
    SEQ_SCATTER_SHUFFLE: "scatter_shuffle", SEQ_GUIDED_REBUILD: "guided_rebuild",
}



@dataclass
class OperatorContext:
    """operators.py:54-66: what an operator may consult besides the solution.
    On the device `pick_mate` draws from the population snapshot and `phi` is
    the kernel's scalarised fitness; here `pick_mate` is called on the host to
    supply apply_sequence's crossover mate, and `phi=None` keeps the
    reference's guided-rebuild fallback to scatter shuffle
    (operators.py:510-512)."""

    problem: object
    cfg: ProblemConfig
    pick_mate: Callable | None = None
    phi: Callable | None = None


@dataclass
class SequenceEntry:
    id: int
    name: str
    fn: Callable | None = None
    weight: float = 1.0
    floor: float = 0.0
    cap: float = math.inf


@dataclass
class CustomOperator:
    """A user operator.  `cuda` is the body of
    `template <class Ctx> __device__ void op(Ctx& ctx)` (see DESIGN.md
    "User operators" for the Ctx API).  `apply` is accepted for source
    compatibility with the reference and ignored."""

    id: int
    name: str
    apply: Callable | None = None
    initial_weight: float = 1.0
    cuda: str | None = None

    def __post_init__(self):
        if self.initial_weight <= 0:
            raise ValueError("initial_weight must be positive")


class SequenceRegistry:
    def __init__(self, entries: list[SequenceEntry]):
        ids = [e.id for e in entries]
        if len(set(ids)) != len(ids):
            raise ValueError("duplicate sequence ids in registry")
        self.entries = list(entries)
        self.normalize()

    def __len__(self):
        return len(self.entries)

    def ids(self) -> list[int]:
        return [e.id for e in self.entries]

    def get(self, seq_id: int) -> SequenceEntry:
        for e in self.entries:
            if e.id == seq_id:
                return e
        raise KeyError(f"sequence id {seq_id} not in registry")

    def normalize(self):
        # builtin sum(): Neumaier-compensated for Python floats (CPython >= 3.12)
        total = sum(e.weight for e in self.entries)
        if total <= 0:
            raise ValueError("registry weights must have positive mass")
        for e in self.entries:
            e.weight /= total

    def total(self) -> float:
        """sum(e.weight ...) exactly as sample_sequence computes it (aos.py:168)."""
        return sum(e.weight for e in self.entries)

    def weights(self):
        return [e.weight for e in self.entries]

    def copy(self) -> "SequenceRegistry":
        out = SequenceRegistry.__new__(SequenceRegistry)
        out.entries = [SequenceEntry(e.id, e.name, e.fn, e.weight, e.floor, e.cap)
                       for e in self.entries]
        return out


def lns_scope(n: int) -> int:
    if n < 1:
        raise ValueError("problem size must be >= 1")
    return max(2, math.ceil(min(0.1 * n, 30.0)))


def sequence_applicable(seq_id: int, cfg: ProblemConfig) -> bool:
    """operators.py:574-597."""
    kind = cfg.encoding.kind
    if seq_id in (SEQ_SWAP, SEQ_INSERT, SEQ_REVERSE, SEQ_OR_OPT, SEQ_THREE_OPT, SEQ_OX_CROSSOVER):
        return kind is EncodingKind.PERMUTATION
    if seq_id in (SEQ_FLIP, SEQ_SEG_FLIP):
        return kind is EncodingKind.BINARY
    if seq_id in (SEQ_RANDOM_RESET, SEQ_SEG_RESET):
        return kind is EncodingKind.INTEGER
    if seq_id == SEQ_UNIFORM_CROSSOVER:
        return kind in (EncodingKind.BINARY, EncodingKind.INTEGER)
    if seq_id == SEQ_ROW_SWAP:
        return cfg.d1 >= 2
    if seq_id in (SEQ_ROW_SPLIT, SEQ_ROW_MERGE):
        return cfg.row_mode is RowModeKind.MULTI_PARTITION
    if seq_id in LNS_IDS:
        return True
    raise KeyError(f"unknown built-in sequence id {seq_id}")


def build_registry(cfg: ProblemConfig, allowed=None) -> SequenceRegistry:
    """Applicable built-ins in id order (operators.py:618-624).  The engine
    passes `allowed` = the problem's device sequences (problem.device_sequences()),
    so the registry holds exactly the operators the device kernel runs."""
    entries = [SequenceEntry(sid, name) for sid, name in BUILTIN_NAMES.items()
               if sequence_applicable(sid, cfg) and (allowed is None or sid in allowed)]
    if not entries:
        raise NotImplementedError("no device operators for this encoding / row mode")
    return SequenceRegistry(entries)


def missing_device_sequences(cfg: ProblemConfig, device: tuple) -> list[int]:
    """Reference sequences for this layout that the device does not run yet."""
    return [sid for sid in BUILTIN_NAMES if sequence_applicable(sid, cfg) and sid not in device]


def validate_custom_id(registry: SequenceRegistry, op: CustomOperator):
    """operators.py:641-648 hard errors."""
    if op.id < CUSTOM_ID_START:
        raise ValueError(f"custom operator id must be >= {CUSTOM_ID_START} (got {op.id}; ids "
                         f"below 32 are built-in, [32, 100) is reserved)")
    if op.id in registry.ids():
        raise ValueError(f"sequence id {op.id} already registered")


def append_custom(registry: SequenceRegistry, op: CustomOperator):
    """operators.py:666-668: append, then renormalise after each registration."""
    registry.entries.append(SequenceEntry(op.id, op.name, None, weight=op.initial_weight))
    registry.normalize()


def apply_sequence(registry: SequenceRegistry, seq_id: int, sol, rng, ctx: OperatorContext):
    """operators.py:627-631: apply exactly one registered operator to `sol` in
    place — on the device (engine.apply_operator_device): a one-lane evolve
    step whose registry holds only this sequence, always accepted.  Draws come
    from a Philox stream keyed by 64 bits of `rng`, not from `rng` itself."""
    registry.get(seq_id)  # KeyError for an unregistered id (operators.py:107-111)
    from .engine import apply_operator_device
    apply_operator_device(registry, seq_id, sol, rng, ctx)


def register_custom(registry: SequenceRegistry, op: CustomOperator, probe, ctx: OperatorContext,
                    probe_rng) -> bool:
    """operators.py:634-669 for CUDA operators: a bad id is a hard error; the
    snippet is compiled by NVRTC together with the operators already
    registered on ctx.problem and probed once on `probe` on the device.  A
    compile error, a device fault or an invalid result excludes it with a
    RuntimeWarning (registry unchanged, returns False); otherwise it is
    appended with its initial weight and the registry renormalised."""
    import warnings
    validate_custom_id(registry, op)
    if not op.cuda:
        warnings.warn(f"custom operator {op.name!r} (id {op.id}) excluded: no CUDA snippet "
                      "(the device engine cannot run Python operators)", RuntimeWarning,
                      stacklevel=2)
        return False
    from .engine import probe_custom_device
    ok, msg = probe_custom_device(ctx.problem, op, probe, probe_rng)
    if not ok:
        warnings.warn(f"custom operator {op.name!r} (id {op.id}) excluded: {msg}", RuntimeWarning,
                      stacklevel=2)
        return False
    append_custom(registry, op)
    return True

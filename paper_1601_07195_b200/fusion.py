"""Gate fusion: the GPU analogue of the paper's cache blocking (mirror of pkg/src/svsim/fusion.py).

Planning is the reference's greedy pass, unchanged in meaning
(fusion.py:71-94): a gate joins the open run iff all its qubits are below the
block exponent l_c.  Execution differs in where the block lives: a fused run
is one ``sv_apply_fused`` launch per (at most 256) gates, each CTA loading a
2^T-amplitude tile (T = 12 or 13, 64-128 KiB) into shared memory once,
applying the whole gate list in order and storing once -- one HBM pass for
the run instead of one per gate.  Results are bit-identical to unfused
execution because every amplitude sees the same pair updates in the same
order.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import _lib
from .circuits import Circuit, GateOp
from .core import LocalState
from .distributed import ScratchPool, apply_op
from .errors import FusionContractError
from .kernels import SERIAL, ThreadPolicy, apply_controlled_raw, apply_single_raw, launch_fused

GPU_MAX_BLOCK_EXPONENT = _lib.SV_FUSED_MAX_TILE


@dataclass(frozen=True)
class FusionConfig:
    """l_c: block exponent (blocks of 2^l_c amplitudes).

    ``passes=True`` (an extension, off by default so plans match the
    reference) replaces block runs by the native pass planner of passes.py:
    l_c then sets the register tile (clamped to [9, 13]).

    ``exact=False`` (with ``passes=True`` only; opt-in) trades bitwise parity for
    fewer operations: consecutive gates on the same qubits multiply into one
    2x2 matrix and stage passes collapse every diagonal gate controlled from
    outside the pass into one per-amplitude factor (k_dstage).  Results then
    match the reference within rounding -- north_star's max-abs <= 1e-12 sqrt(G)
    bound for fused gates -- instead of bit for bit."""

    l_c: int
    enabled: bool = True
    passes: bool = False
    exact: bool = True

    def __post_init__(self):
        if self.l_c < 1:
            raise ValueError("block exponent must be >= 1")
        if not self.exact and not self.passes:
            raise ValueError("exact=False needs passes=True (the tolerance mode is a pass-planner mode)")


def default_block_exponent(llc_bytes: int, m: int) -> int:
    """Reference rule (fusion.py:33-42): largest l_c whose block fills at most half the cache."""
    if llc_bytes < 64:
        raise ValueError("cache size implausibly small")
    return min(m, max(1, (llc_bytes // 32).bit_length() - 1))


def gpu_block_exponent(m: int) -> int:
    """Largest block one CTA keeps resident in shared memory (2^13 x 16 B = 128 KiB)."""
    return min(m, GPU_MAX_BLOCK_EXPONENT)


@dataclass(frozen=True)
class FusedBlockRun:
    gates: tuple[GateOp, ...]


@dataclass(frozen=True)
class PassThrough:
    gate: GateOp


@dataclass
class FusionPlan:
    l_c: int
    segments: list = field(default_factory=list)
    passes: bool = False
    exact: bool = True

    def flatten(self) -> list[GateOp]:
        out: list[GateOp] = []
        for seg in self.segments:
            if isinstance(seg, FusedBlockRun):
                out.extend(seg.gates)
            else:
                out.append(seg.gate)
        return out


def plan_fusion(circuit: Circuit, config: FusionConfig) -> FusionPlan:
    """Greedy maximal runs in circuit order, no reordering (fusion.py:71-94)."""
    plan = FusionPlan(config.l_c, passes=config.enabled and config.passes, exact=config.exact or not config.enabled)
    if plan.passes:  # the pass planner needs m; execute_plan cuts the passes
        plan.segments = [PassThrough(op) for op in circuit]
        return plan
    run: list[GateOp] = []
    for op in circuit:
        if config.enabled and op.max_qubit() < config.l_c:
            run.append(op)
            continue
        if run:
            plan.segments.append(FusedBlockRun(tuple(run)))
            run = []
        plan.segments.append(PassThrough(op))
    if run:
        plan.segments.append(FusedBlockRun(tuple(run)))
    return plan


def run_fused(state: LocalState, gates, l_c: int) -> int:
    """Execute one FusedBlockRun on the device; returns the number of HBM passes.

    Gates whose qubits fit a shared-memory tile go out in fused launches
    (split at SV_FUSED_MAX_GATES); with l_c beyond the tile limit, gates on
    qubits >= 13 run as single passes in order between them.
    """
    gates = list(gates)
    for op in gates:
        if op.max_qubit() >= l_c:
            raise FusionContractError(f"gate on qubits {op.qubits()} exceeds block exponent {l_c}")
    passes = 0
    group: list[GateOp] = []

    def flush() -> None:
        nonlocal passes, group
        if group:
            lg = max(op.max_qubit() for op in group) + 1
            launch_fused(state.amps, group, lg)
            passes += -(-len(group) // _lib.SV_FUSED_MAX_GATES)
            group = []

    for op in gates:
        if op.max_qubit() < GPU_MAX_BLOCK_EXPONENT:
            group.append(op)
            continue
        flush()
        if op.control is None:
            apply_single_raw(state.amps, op.target, op.gate)
        else:
            apply_controlled_raw(state.amps, op.control, op.target, op.gate)
        passes += 1
    flush()
    return passes


def execute_plan(state: LocalState, plan: FusionPlan, policy: ThreadPolicy = SERIAL, transport=None, *,
                 chunk_amps: int | None = None, scratch: ScratchPool | None = None) -> None:
    """Fused runs as tile passes, pass-throughs through apply_op (fusion.py:97-135)."""
    if plan.passes:
        from .passes import execute_pass, plan_passes, tile_for

        tile = tile_for(plan.l_c, state.layout.m)
        for p in plan_passes(plan.flatten(), state.layout.m, tile, exact=plan.exact):
            execute_pass(state, p, transport, tile=tile)
        return
    if plan.l_c > state.layout.m:
        raise FusionContractError(f"block exponent {plan.l_c} exceeds local qubit count m={state.layout.m}")
    for seg in plan.segments:
        if isinstance(seg, PassThrough):
            apply_op(state, seg.gate, transport, policy=policy, chunk_amps=chunk_amps, scratch=scratch)
        else:
            run_fused(state, seg.gates, plan.l_c)

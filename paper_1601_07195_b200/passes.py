"""Pass fusion: the native planner behind ``FusionConfig(passes=True)``.

The reference fuses only runs of gates whose qubits all sit below l_c
(fusion.py:71-94); every other gate is its own sweep over memory.  With
``passes=True`` the circuit is cut into as few HBM passes as the kernels
allow, without reordering any gate:

* ``local`` pass -- a maximal run of gates with a local target (controls
  anywhere; a control in the rank bits turns into "uncontrolled" or "skip" on
  this rank).  Executed by ``sv_apply_gates``: register-tiled runs for
  targets below bit 4 of the tile (2^12) plus up to eight gathered higher qubits,
  multi-target stage passes for runs whose targets lie in at most four qubits
  (four transform stages H(k), R(k, c) for all c are ONE pass), single-gate
  kernels otherwise -- whichever covers the run more cheaply (svb200.cu
  ``next_group``).
* ``global_stage`` -- a run of gates sharing one global target: ONE fused
  NVLink exchange applies them all (``sv_exchange_stage``).
* ``global_gate`` -- a lone global-target gate: the reference-equivalent
  exchange (``apply_global``, per-gate traffic contract preserved).

Results are bit-identical to the reference's unfused execution: every pair
sees the same updates in the same order, and the structure-specialised
updates (diagonal / phase / real / Hadamard-like gates) are exact -- they
differ from mix() only in zero signs, and any zero in a pass's final values
sends that group through an exact replay (svb200.cu "speculative pair updates").

``exact=False`` (FusionConfig(passes=True, exact=False), the tolerance mode):
before planning, a gate merges into the latest earlier gate that acts on
exactly its qubits in the same roles when nothing in between touched them (the
product of the two 2x2 matrices; ``merge_gates``); a run of local gates is
reordered past commuting gates when that saves HBM passes (``schedule_gates``);
and stage passes run
k_dstage, which folds every diagonal gate controlled from outside the pass
into one per-amplitude factor.  Values agree with the reference within
rounding (north_star: max-abs <= 1e-12 sqrt(G), fused gates included), not bit
for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .circuits import GateOp
from .distributed import _CUDA, GateAction, _check_transport, _fence, apply_global, fingerprint
from .perfmodel import BoundCase
from .errors import LayoutError, TransportError
from .kernels import GateMatrix, _as_gate


LOCAL_KINDS = ("local_tile", "local_stage", "local_gate", "local_low", "local_stage2")


@dataclass(frozen=True)
class Pass:
    kind: str                # local_tile | local_stage | local_gate | local_low (tolerance) | global_*
    gates: tuple[GateOp, ...]
    target: int | None = None
    exact: bool = True       # False: tolerance mode (stage passes through k_dstage)

    @property
    def local(self) -> bool:
        return self.kind in LOCAL_KINDS


def merge_gates(gates) -> list[GateOp]:
    """Tolerance mode: a gate multiplies into the latest earlier gate with the same target and
    control when no gate in between touched either qubit (those gates commute with it), so
    e.g. repeated rotations of one qubit become one 2x2 matrix.  Pure host arithmetic."""
    out: list[GateOp] = []
    last: dict[int, int] = {}
    for op in gates:
        qs = op.qubits()
        j = last.get(qs[0], -1)
        if j >= 0 and all(last.get(q, -1) == j for q in qs):
            prev = out[j]
            if prev.target == op.target and prev.control == op.control:
                mat = np.asarray(_as_gate(op.gate).mat) @ np.asarray(_as_gate(prev.gate).mat)
                out[j] = GateOp(GateMatrix.unchecked(mat), op.target, op.control, prev.name)
                continue
        out.append(op)
        for q in qs:
            last[q] = len(out) - 1
    return out


def _is_diagonal(op: GateOp) -> bool:
    mat = np.asarray(_as_gate(op.gate).mat)
    return mat[0, 1] == 0 and mat[1, 0] == 0


def schedule_gates(ops, tile: int, gather: int = _lib.SV_TILE_GATHER) -> list[GateOp]:
    """Tolerance mode: reorder a run of local gates, moving a gate only past gates it commutes
    with, so that consecutive gates share a register tile (targets below ``tile - gather`` plus
    at most ``gather`` other qubits) and the native planner needs fewer HBM passes.

    Two gates commute when on every qubit they share both act diagonally -- as a control, or as
    the target of a diagonal matrix -- so the order kept is: on each qubit, a non-diagonal gate
    stays behind everything earlier and ahead of everything later.  Within a tile the gates are
    grouped four target qubits at a time, highest qubits first (the register sets of k_tile;
    the first set is the layout of the global load).  Pure host code, deterministic: every
    rank derives the same order."""
    ops = list(ops)
    n = len(ops)
    low = max(tile - gather, 0)
    succ: list[list[int]] = [[] for _ in range(n)]
    indeg = [0] * n
    last_t: dict[int, int] = {}
    since: dict[int, list[int]] = {}
    for i, op in enumerate(ops):
        roles = {op.target: _is_diagonal(op)}
        if op.control is not None:
            roles[op.control] = True
        deps = set()
        for q, diag in roles.items():
            if q in last_t:
                deps.add(last_t[q])
            if diag:
                since.setdefault(q, []).append(i)
            else:
                deps.update(since.get(q, ()))
                last_t[q] = i
                since[q] = []
        deps.discard(i)
        for d in deps:
            succ[d].append(i)
        indeg[i] = len(deps)
    ready = sorted(i for i in range(n) if indeg[i] == 0)
    order: list[int] = []
    while ready:
        targets: set[int] = set()
        chosen: list[int] = []
        while True:
            take = [g for g in ready if ops[g].target < low or ops[g].target in targets]
            if take:
                for g in take:
                    ready.remove(g)
                    chosen.append(g)
                    for v in succ[g]:
                        indeg[v] -= 1
                        if indeg[v] == 0:
                            ready.append(v)
                ready.sort()
                continue
            if len(targets) == gather or not ready:
                break
            count: dict[int, int] = {}
            for g in ready:
                count[ops[g].target] = count.get(ops[g].target, 0) + 1
            best = max(count, key=lambda t: (count[t], -min(g for g in ready if ops[g].target == t)))
            targets.add(best)
        # inside the pass: register sets of four gathered qubits, highest first, low qubits last
        rank = {t: k for k, t in enumerate(sorted(targets, reverse=True))}
        key = {g: (rank[ops[g].target] // 4 if ops[g].target in rank else len(rank)) for g in chosen}
        pos = {g: k for k, g in enumerate(chosen)}
        inside = set(chosen)
        deg = {g: 0 for g in chosen}
        for g in chosen:
            for v in succ[g]:
                if v in inside:
                    deg[v] += 1
        avail = [g for g in chosen if deg[g] == 0]
        while avail:
            g = min(avail, key=lambda x: (key[x], pos[x]))
            avail.remove(g)
            order.append(g)
            for v in succ[g]:
                if v in inside:
                    deg[v] -= 1
                    if deg[v] == 0:
                        avail.append(v)
    assert len(order) == n
    return [ops[g] for g in order]


def _gate_class(op: GateOp) -> str:
    """general / diagonal / real / hadamard-like, as the native planner's cost model sees a gate."""
    mat = np.asarray(_as_gate(op.gate).mat)
    if mat[0, 1] == 0 and mat[1, 0] == 0:
        return "diag"
    if np.any(mat.imag != 0):
        return "general"
    return "hlike" if mat[0, 0] == mat[0, 1] == mat[1, 0] == -mat[1, 1] else "real"


_TILE_COST = {"general": 1.15, "diag": 0.45, "real": 0.75, "hlike": 0.55}
_STAGE_COST = {"general": 0.9, "diag": 0.02, "real": 0.55, "hlike": 0.35}


def plan_cost(plan) -> float:
    """Estimated milliseconds at 2^30 amplitudes of a tolerance-mode plan of local passes: the
    native planner's model (svb200.cu next_group: a pass costs max(5, its gates' FP64 time); a
    low-bit pass 5.5, a mostly diagonal two-phase pass 7).  Only used to choose between the
    circuit's own order and the scheduled one."""
    total = 0.0
    for p in plan:
        if p.kind == "local_low":
            total += 5.5
        elif p.kind == "local_stage2":
            total += max(7.0, sum(_STAGE_COST[_gate_class(op)] for op in p.gates))
        elif p.kind == "local_stage":
            total += max(5.0, sum(_STAGE_COST[_gate_class(op)] * (0.5 if op.control is not None else 1.0)
                                  for op in p.gates))
        elif p.kind == "local_tile":
            total += max(5.0, sum(_TILE_COST[_gate_class(op)] for op in p.gates))
        else:
            total += 5.0 * len(p.gates)
    return total


def plan_passes(gates, m: int, tile: int = 0, exact: bool = True) -> list[Pass]:
    """Cut a gate sequence into HBM passes -- a pure function of the gates, m and the tile,
    so every rank derives the same list (the collective fences line up).

    Local targets: the native planner's groups (``sv_plan_gates``): a register-tiled
    ``local_tile`` pass, a multi-target ``local_stage`` pass, or a lone ``local_gate``.
    Global targets: a run sharing the target is one ``global_stage`` exchange.  This is the
    grouping ``sv_apply_gates`` applies natively, exposed so each pass can be
    timed and recorded on its own.  exact=False: the tolerance mode (``merge_gates``
    first, stage passes planned and run for k_dstage)."""
    gates = list(gates) if exact else merge_gates(gates)
    out: list[Pass] = []
    i, n = 0, len(gates)
    while i < n:
        t = gates[i].target
        j = i + 1
        if t >= m:
            while j < n and gates[j].target == t and j - i < _lib.SV_STAGE_MAX_GATES:
                j += 1
            out.append(Pass("global_stage" if j - i > 1 else "global_gate", tuple(gates[i:j]), t, exact))
        else:
            while j < n and gates[j].target < m:
                j += 1
            local = _plan_local(gates[i:j], m, tile, exact)
            if not exact and tile >= 9 and len(local) > 1:
                # the commutation-aware order, when the native planner's passes get cheaper with it
                again = _plan_local(schedule_gates(gates[i:j], tile), m, tile, exact)
                if plan_cost(again) < 0.98 * plan_cost(local):
                    local = again
            out.extend(local)
        i = j
    return out


_GROUP_KIND = {_lib.SV_GROUP_GATES: "local_gate", _lib.SV_GROUP_TILE: "local_tile",
               _lib.SV_GROUP_STAGE: "local_stage", _lib.SV_GROUP_LOW: "local_low",
               _lib.SV_GROUP_STAGE2: "local_stage2"}
_KIND_GROUP = {v: k for k, v in _GROUP_KIND.items()}


def _plan_local(ops, m: int, tile: int, exact: bool = True) -> list[Pass]:
    """Split a run of local-target gates into launch groups with the native planner
    (sv_plan_gates, the one sv_apply_gates executes).  Rank-bit controls only decide
    per rank whether a gate applies, so they are planned as uncontrolled."""
    import ctypes

    arr = (_lib.SvGate * len(ops))()
    for k, op in enumerate(ops):
        arr[k].target = op.target
        arr[k].control = -1 if op.control is None or op.control >= m else op.control
        arr[k].q[:] = list(_as_gate(op.gate).qbuf())
    ends = (ctypes.c_int32 * len(ops))()
    kinds = (ctypes.c_int32 * len(ops))()
    ng = _lib.load().sv_plan_gates_ex(m, arr, len(ops), int(tile), 0 if exact else _lib.SV_FLAG_TOLERANCE,
                                      ends, kinds, len(ops))
    if ng < 0:
        _lib.check(ng)
    out, start = [], 0
    for g in range(ng):
        out.append(Pass(_GROUP_KIND[kinds[g]], tuple(ops[start:ends[g]]), ops[start].target, exact))
        start = ends[g]
    return out


def _resolve_rank_controls(ops, layout) -> list[GateOp]:
    """Gates whose control is a rank bit become uncontrolled (bit set) or vanish (bit clear)."""
    out = []
    for op in ops:
        c = op.control
        if c is not None and c >= layout.m:
            if (layout.rank >> (c - layout.m)) & 1:
                out.append(GateOp(op.gate, op.target, None, op.name))
        else:
            out.append(op)
    return out


def execute_pass(state, p: Pass, transport=None, *, tile: int = 0, executor=None) -> None:
    lay = state.layout
    ex = executor or (transport.executor if transport is not None else _CUDA)
    if p.local:
        ops = _resolve_rank_controls(p.gates, lay)
        if ops:
            if p.exact:
                ex.local_gates(state, ops, tile, group=_KIND_GROUP[p.kind])
            else:
                ex.local_gates(state, ops, tile, group=_KIND_GROUP[p.kind], exact=False)
        return
    if transport is None:
        raise LayoutError(f"gate on qubit {p.target} >= m={lay.m} requires a transport")
    if p.kind == "global_gate":
        op = p.gates[0]
        apply_global(state, op.target, op.control, op.gate, transport, executor=executor)
        return
    _check_transport(transport, lay)
    tag = transport.fresh_tag()
    transport.ensure_registered(state)
    bit = p.target - lay.m
    partner = lay.rank ^ (1 << bit)
    zero = ((lay.rank >> bit) & 1) == 0
    ops = [GateOp(_as_gate(op.gate), op.target, op.control, op.name)
           for op in _resolve_rank_controls(p.gates, lay)]
    fp = fingerprint(tag, p.target, len(p.gates), 0x57A6E)
    try:
        _fence(transport, state, fp)
        if ops and getattr(transport, "data_plane", "ipc") in ("nccl", "ce"):
            for op in ops:  # staged planes: one chunked exchange per gate of the stage
                act = GateAction("exchange", BoundCase.SINGLE_REMOTE, op.target, op.control, partner=partner,
                                 own_is_zero=zero, c_local=-1 if op.control is None else op.control)
                moved = transport.staged_exchange(state, act, op.gate)
                transport.count(moved, moved)
        elif ops:
            ex.exchange_stage(state, transport.peer_pointer(state, partner), zero, ops)
            transport.count(1 << (lay.m + 4), 1 << (lay.m + 4))
        _fence(transport, state, fp)
    except TransportError:
        state.corrupt = True
        raise
    except Exception as exc:
        state.corrupt = True
        raise TransportError(f"stage exchange for qubit {p.target} failed: {exc}") from exc
    except BaseException:
        state.corrupt = True
        raise


def tile_for(l_c: int, m: int) -> int:
    """Tile exponent of the register-tiled kernel for a FusionConfig block exponent."""
    t = min(l_c, m, _lib.SV_FUSED_MAX_TILE)
    return t if t >= 9 else 0

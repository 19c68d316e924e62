"""Communication-avoiding execution: swap global and local qubits instead of exchanging
for every gate on a global qubit (PAPER.md:478 names it as future work).

The reference runs every gate on a global qubit as an in-place pairwise exchange
(distributed.py:314-422): 2^(m+4) bytes per direction per gate.  Here a gate whose
target sits on a global (rank) bit first swaps that bit with a local bit
(``sv_swap_global``: 2^(m+3) bytes per direction, once); the gate -- and every later
gate on that logical qubit until it is swapped back -- then runs locally in HBM.

The logical -> physical qubit map is kept as a set of disjoint global<->local
transpositions, so it is undone by one swap per transposition:

* a gate on a logical qubit whose home is local but which sits on a global bit (it was
  a victim) swaps back home -- that restores both qubits of the transposition;
* a gate on a logical global qubit at home picks a victim among the local qubits that
  are at home and not used by the gate, the one whose next use lies furthest ahead
  (Belady), and swaps with it.

The plan is a pure function of (gates, n, m), so every rank derives the same swaps and
the fences line up.  Swaps only move amplitudes and the gates see exactly the
reference's operand pairs, so results -- after the final restoring swaps -- are
bit-identical to the in-place exchange.  Control qubits on global bits are handled by
the usual rank predicates (cases 4 and 6 of perfmodel.py:30-38).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .circuits import Circuit, GateOp
from .errors import LayoutError, TransportError


@dataclass
class QubitMap:
    """pos[logical] = physical bit, occ[physical] = logical qubit."""

    n: int
    pos: list[int] = field(default_factory=list)
    occ: list[int] = field(default_factory=list)

    def __post_init__(self):
        if not self.pos:
            self.pos = list(range(self.n))
            self.occ = list(range(self.n))

    def swap(self, a: int, b: int) -> None:
        la, lb = self.occ[a], self.occ[b]
        self.occ[a], self.occ[b] = lb, la
        self.pos[la], self.pos[lb] = b, a

    @property
    def identity(self) -> bool:
        return all(p == q for q, p in enumerate(self.pos))


@dataclass(frozen=True)
class Swap:
    global_bit: int  # physical global qubit G >= m
    local_bit: int   # physical local qubit l < m


def plan_remapped(gates, n: int, m: int, restore: bool = True, qmap: QubitMap | None = None):
    """Items in execution order: lists of PHYSICAL GateOps and Swap records.  Every target
    is local except when all local qubits are already displaced (more global than local
    qubits); such a gate runs as the reference's in-place exchange.  Returns (items, map)."""
    gates = list(gates)
    qm = qmap or QubitMap(n)
    uses: dict[int, list[int]] = {}
    for i, op in enumerate(gates):
        for q in op.qubits():
            uses.setdefault(q, []).append(i)
    nxt = {q: 0 for q in uses}

    def next_use(q: int, i: int) -> float:
        lst = uses.get(q, [])
        k = nxt.get(q, 0)
        while k < len(lst) and lst[k] < i:
            k += 1
        nxt[q] = k
        return lst[k] if k < len(lst) else float("inf")

    items: list = []
    cur: list[GateOp] = []
    for i, op in enumerate(gates):
        t = qm.pos[op.target]
        if t >= m:
            if op.target < m:  # a displaced local qubit: swap back home
                victim = op.target
            else:
                busy = {qm.pos[q] for q in op.qubits()}
                cands = [b for b in range(m) if qm.occ[b] == b and b not in busy]
                if not cands:  # every local qubit is displaced (more global than local qubits):
                    c = None if op.control is None else qm.pos[op.control]  # exchange in place
                    cur.append(GateOp(op.gate, t, c, op.name))
                    continue
                victim = max(cands, key=lambda b: (next_use(b, i + 1), b))
            if cur:
                items.append(cur)
                cur = []
            items.append(Swap(t, victim))
            qm.swap(t, victim)
        c = None if op.control is None else qm.pos[op.control]
        cur.append(GateOp(op.gate, qm.pos[op.target], c, op.name))
    if cur:
        items.append(cur)
    if restore:
        for g in range(m, n):
            if qm.occ[g] != g:
                sw = Swap(g, qm.pos[g])
                items.append(sw)
                qm.swap(sw.global_bit, sw.local_bit)
    return items, qm


def swap_global(state, sw: Swap, transport, executor=None) -> None:
    """One rank's side of a global<->local swap, between two partner fences.  Peer-mapped
    planes run k_swap_global on the partner's slice; the NCCL plane sends the moving half
    (bit l = 1 - b) and receives the partner's in its place, chunk by chunk."""
    from .distributed import _check_transport, _fence, fingerprint

    lay = state.layout
    _check_transport(transport, lay)
    if not (lay.m <= sw.global_bit < lay.n and 0 <= sw.local_bit < lay.m):
        raise LayoutError(f"swap ({sw.global_bit}, {sw.local_bit}) is not global <-> local for m={lay.m}")
    tag = transport.fresh_tag()
    transport.ensure_registered(state)
    ex = executor or transport.executor
    bit = sw.global_bit - lay.m
    partner = lay.rank ^ (1 << bit)
    b = (lay.rank >> bit) & 1
    fp = fingerprint(tag, sw.global_bit, sw.local_bit, 0x5A9)
    try:
        _fence(transport, state, fp)
        if getattr(transport, "mapped", True):
            ex.swap_global(state, transport.peer_pointer(state, partner), b == 0, sw.local_bit)
        else:
            _swap_staged(transport, state, sw.local_bit, b, partner)
        transport.count(1 << (lay.m + 3), 1 << (lay.m + 3))
        _fence(transport, state, fp)
    except TransportError:
        state.corrupt = True
        raise
    except Exception as exc:
        state.corrupt = True
        raise TransportError(f"swap of qubits ({sw.global_bit}, {sw.local_bit}) failed: {exc}") from exc
    except BaseException:
        state.corrupt = True
        raise


def _swap_staged(fabric, state, l: int, b: int, partner: int) -> None:
    """The swap over send/recv: own elements with bit l = 1 - b <-> the partner's with bit l = b,
    in the same (row, column) order on both sides; pieces of at most chunk_amps elements."""
    import torch.distributed as dist

    whole = fabric.executor.tensor(state)
    sel = whole.view(-1, 2, 1 << l)[:, 1 - b, :]
    rows, width = sel.shape
    chunk = max(1, fabric.chunk_amps)
    if width >= chunk:
        pieces = [sel[r, c0:c0 + chunk] for r in range(rows) for c0 in range(0, width, chunk)]
    else:
        per = max(1, chunk // width)
        pieces = [sel[r0:r0 + per] for r0 in range(0, rows, per)]
    peer = fabric._global_peer(partner)
    dev = fabric.executor.buffer_device(state)
    for piece in pieces:
        out = piece.contiguous().view(-1)
        inb = fabric.scratch.take(out.numel(), device=dev)
        try:
            if fabric.fence_mode == "stream":
                for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, out, peer, fabric.group),
                                                 dist.P2POp(dist.irecv, inb, peer, fabric.group)]):
                    w.wait()
            elif b == 0:  # blocking transport: the zero side sends first
                fabric._send(out, peer)
                fabric._recv(inb, peer)
            else:
                fabric._recv(inb, peer)
                fabric._send(out, peer)
            piece.copy_(inb.view(piece.shape))
        finally:
            fabric.scratch.give(inb)


def run_circuit_remapped(states, circuit: Circuit, transports, *, fusion=None, restore: bool = True,
                         qmap: QubitMap | None = None, executor=None) -> QubitMap:
    """Run ``circuit`` with global<->local swaps instead of per-gate exchanges.

    ``states`` / ``transports``: this rank's state and fabric (one process per GPU), or
    lists of every rank's (in-process ranks, InprocFabric), run rank by rank per step.
    With restore=True the final map is the identity and the slices hold exactly what
    ``run_circuit`` would have produced; otherwise pass the returned map back in (qmap=)
    to continue, and restore later with ``restore_map``."""
    from .engine import run_circuit

    if not isinstance(states, (list, tuple)):
        states, transports = [states], [transports]
    lay = states[0].layout
    if circuit.n != lay.n:
        raise LayoutError(f"circuit has {circuit.n} qubits, state has {lay.n}")
    if lay.p == 0:
        for st, tr in zip(states, transports):
            run_circuit(st, circuit, tr, fusion=fusion)
        return qmap or QubitMap(lay.n)
    items, qm = plan_remapped(circuit.gates, lay.n, lay.m, restore, qmap)
    for item in items:
        if isinstance(item, Swap):
            for st, tr in zip(states, transports):
                swap_global(st, item, tr, executor)
        elif executor is not None:  # a non-CUDA executor (tests): the pass machinery drives it
            from .passes import execute_pass, plan_passes

            for pz in plan_passes(item, lay.m, 0):
                for st, tr in zip(states, transports):
                    execute_pass(st, pz, tr, executor=executor)
        else:
            sub = Circuit(lay.n, item)
            if len(states) == 1:
                run_circuit(states[0], sub, transports[0], fusion=fusion)
            else:
                from .engine import run_circuit_inproc

                run_circuit_inproc(states, sub, transports, fusion=fusion)
    return qm


def restore_map(states, qmap: QubitMap, transports) -> None:
    """Undo the transpositions of ``qmap`` (one swap each)."""
    if not isinstance(states, (list, tuple)):
        states, transports = [states], [transports]
    m = states[0].layout.m
    for g in range(m, qmap.n):
        if qmap.occ[g] != g:
            sw = Swap(g, qmap.pos[g])
            for st, tr in zip(states, transports):
                swap_global(st, sw, tr)
            qmap.swap(sw.global_bit, sw.local_bit)

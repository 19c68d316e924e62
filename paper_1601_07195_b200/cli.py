"""Command line: run circuit files and benchmark sweeps on B200s.

Mirrors the reference's CLI (pkg/src/svsim/cli.py:1-585): the subcommands
``run``, ``gate-bench``, ``qft-bench`` and ``bounds``, the circuit-file format
(circuitfile.py), CSV / JSON output (``"schema": 1``) and the exit codes
0 ok, 2 usage, 3 circuit parse error, 4 resource refusal, 5 transport failure.

What changes is the machine underneath:
  * one process per GPU.  Under ``torchrun`` (WORLD_SIZE = 2^p) each rank holds
    its 2^(n-p) slice in HBM and global-qubit gates run the NVLink exchange
    (NvlinkFabric over NCCL).  Without torchrun, ``--ranks R`` keeps all R rank
    slices on one GPU in this process (InprocFabric, the reference's inproc
    transport); ``--transport tcp`` is gone (usage error);
  * timings are CUDA events on the launch stream (max over ranks), not
    perf_counter;
  * ``--fusion`` also accepts ``passes`` (the native pass planner);
    ``--threads`` is accepted and ignored (the CUDA grid replaces ThreadPolicy).

    python -m paper_1601_07195_b200 run circuit.qc --format json
    torchrun --nproc-per-node 8 -m paper_1601_07195_b200 gate-bench --qubits 36
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import sys
from pathlib import Path

import numpy as np

from .circuitfile import parse_circuit_file
from .circuits import Circuit, GateOp, build_iqft, build_qft, random_unitary
from .core import AMP_BYTES, Layout, LocalState, global_norm_sq, init_basis_state, probability_of_bit
from .distributed import DEFAULT_CHUNK_BYTES, GATHER_MAX_QUBITS, InprocFabric, NvlinkFabric, gather_full_state
from .errors import CircuitParseError, FusionContractError, LayoutError, ResourceError, TransportError
from .fusion import FusionConfig
from .perfmodel import BoundCase, MachineParams, b200_params, classify_case, lower_bound_seconds, traffic_bytes

MEMORY_FRACTION = 0.9
HBM_BYTES = 180e9  # one B200 (used when no device is visible to size the guard)


# ---------------------------------------------------------------- session: ranks and devices


class Session:
    """The ranks this process drives: its own (torchrun) or all of them (in-process)."""

    def __init__(self, ranks: int, transport: str, diagonal_local: bool = False):
        if transport not in ("inproc", "nvlink"):
            raise ValueError(f"--transport {transport!r}: this build runs 'inproc' (one GPU) or under torchrun")
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if ranks < 1 or ranks & (ranks - 1):
            raise ValueError(f"--ranks must be a power of two, got {ranks}")
        self.world = world
        self.rank = int(os.environ.get("RANK", "0"))
        if world > 1 and ranks not in (1, world):
            raise ValueError(f"--ranks {ranks} does not match WORLD_SIZE {world}")
        self.ranks = world if world > 1 else ranks
        self.p = self.ranks.bit_length() - 1
        self.inproc = world == 1 and self.ranks > 1
        self.diagonal_local = diagonal_local
        self.fabric = None
        self.dist = None

    def start(self):
        import torch

        if not torch.cuda.is_available():
            raise ResourceError("no CUDA device: the gate kernels run on B200s only (no CPU path)")
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        self.device = torch.device("cuda", local)
        if self.world > 1:
            import torch.distributed as dist

            dist.init_process_group("nccl", device_id=self.device)
            self.dist = dist
            self.fabric = NvlinkFabric(diagonal_local=self.diagonal_local)
        return self

    def states(self, n: int, basis: int = 0) -> list[LocalState]:
        rs = range(self.ranks) if self.inproc else [self.rank]
        return [init_basis_state(Layout(n, self.p, r), basis, device=self.device) for r in rs]

    def fabrics(self, states):
        return InprocFabric.group(states) if self.inproc else [self.fabric]

    def run(self, states, circuit, fusion, chunk_amps, record=False):
        from .engine import run_circuit, run_circuit_inproc

        if self.inproc:
            return run_circuit_inproc(states, circuit, self.fabrics(states), fusion=fusion, chunk_amps=chunk_amps,
                                      record=record)
        return run_circuit(states[0], circuit, self.fabric, fusion=fusion, chunk_amps=chunk_amps, record=record)

    def timed(self, fn) -> float:
        """Device seconds of fn() on the current stream, max over ranks."""
        import torch

        self.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        sec = s.elapsed_time(e) * 1e-3
        if self.dist is not None:
            t = torch.tensor([sec], dtype=torch.float64, device=self.device)
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
            sec = float(t.item())
        return max(sec, 1e-9)

    def barrier(self):
        import torch

        torch.cuda.synchronize()
        if self.dist is not None:
            self.dist.barrier()

    def summary(self, states, n: int):
        """(norm, per-qubit P(1), top-8 amplitudes or None) on rank 0."""
        import torch

        if self.inproc:  # the whole register is on this device: read it as one slice
            whole = LocalState(Layout(n), torch.cat([s.amps for s in states]))
            states, fab = [whole], None
        else:
            fab = self.fabric
        st = states[0]
        norm = global_norm_sq(st, fab)
        probs = [probability_of_bit(st, q, fab) for q in range(n)]
        top = None
        if n <= GATHER_MAX_QUBITS:
            full = gather_full_state(st, fab)
            if full is not None:
                order = np.argsort(np.abs(full))[::-1][:8]
                top = [{"index": int(i), "re": float(full[i].real), "im": float(full[i].imag),
                        "prob": float(abs(full[i]) ** 2)} for i in order]
        return norm, probs, top

    def close(self):
        if self.fabric is not None:
            self.fabric.close()
        if self.dist is not None:
            self.dist.destroy_process_group()


def check_memory(n: int, p: int, inproc: bool, chunk_bytes: int) -> None:
    """Refuse runs whose slices (plus a staging chunk) would not fit the device."""
    slices_here = (1 << p) if inproc else 1
    need = slices_here * (1 << (n - p)) * AMP_BYTES + 2 * chunk_bytes
    cap = HBM_BYTES
    try:
        import torch

        if torch.cuda.is_available():
            cap = torch.cuda.mem_get_info()[0]
    except Exception:  # noqa: BLE001 -- sizing only
        pass
    if need > MEMORY_FRACTION * cap:
        raise ResourceError(f"run needs about {need} device bytes but only {int(MEMORY_FRACTION * cap)} "
                            f"of {int(cap)} may be used")


def fusion_config(spec: str | None, m: int) -> FusionConfig | None:
    if spec is None or spec == "off":
        return None
    if spec == "passes":
        return FusionConfig(l_c=min(12, m), passes=True)
    try:
        l_c = int(spec)
    except ValueError:
        raise ValueError(f"--fusion expects an integer block exponent, 'passes' or 'off', got {spec!r}") from None
    if l_c > m:
        raise FusionContractError(f"--fusion {l_c} exceeds local qubit count m={m}")
    return FusionConfig(l_c=l_c)


def chunk_amps(nbytes: int | None) -> int | None:
    if nbytes is None:
        return None
    if nbytes < AMP_BYTES:
        raise ValueError(f"--chunk-bytes must be at least {AMP_BYTES}")
    return 1 << ((nbytes // AMP_BYTES).bit_length() - 1)


def parse_range(spec: str, lo_min: int, hi_max: int, flag: str) -> tuple[int, int]:
    try:
        lo, hi = (int(x) for x in spec.split(":", 1))
    except ValueError:
        raise ValueError(f"{flag} expects 'lo:hi', got {spec!r}") from None
    if not lo_min <= lo <= hi <= hi_max:
        raise ValueError(f"{flag} range {lo}:{hi} outside [{lo_min}, {hi_max}]")
    return lo, hi


def emit(rows: list[dict], columns: list[str], meta: dict, args) -> None:
    if args.format == "json":
        text = json.dumps({"schema": 1, **meta, "rows": rows}, indent=2)
    else:
        buf = io.StringIO()
        buf.writelines(f"# {k}={v}\n" for k, v in meta.items() if not isinstance(v, (list, dict)))
        w = csv.DictWriter(buf, fieldnames=columns, extrasaction="ignore")
        w.writeheader()
        w.writerows(rows)
        text = buf.getvalue().rstrip("\n")
    if args.out:
        Path(args.out).write_text(text + "\n", encoding="utf-8")
    else:
        print(text)


def _session(args, n_min: int) -> Session:
    sess = Session(args.ranks, args.transport, getattr(args, "diagonal_local", False))
    if sess.p >= n_min:
        raise LayoutError(f"{sess.ranks} ranks need more than {n_min} qubits")
    return sess


# ---------------------------------------------------------------- commands


def cmd_run(args) -> int:
    circuit = parse_circuit_file(args.circuit)
    n = circuit.n
    sess = _session(args, n)
    fusion = fusion_config(args.fusion, n - sess.p)
    ca = chunk_amps(args.chunk_bytes)
    check_memory(n, sess.p, sess.inproc, args.chunk_bytes or DEFAULT_CHUNK_BYTES)
    sess.start()
    try:
        states = sess.states(n, args.initial)
        records = sess.run(states, circuit, fusion, ca, record=True)
        norm, probs, top = sess.summary(states, n)
    finally:
        sess.close()
    if sess.rank != 0:
        return 0
    meta = {"command": "run", "circuit": str(args.circuit), "n": n, "p": sess.p, "threads": args.threads,
            "fusion": args.fusion or "off", "norm": norm, "probabilities": probs, "top_amplitudes": top,
            "timing": "CUDA events, device seconds"}
    if args.format == "csv":
        meta["probabilities"] = " ".join(f"{q}:{v:.6f}" for q, v in enumerate(probs))
        meta.pop("top_amplitudes")
    rows = [{"gate": r.index, "kind": r.kind, "qubits": "/".join(map(str, r.qubits)), "case": r.case.case_id,
             "seconds": f"{r.seconds:.6e}", "bytes_moved": r.bytes_moved, "gate_count": r.gate_count}
            for r in records]
    emit(rows, ["gate", "kind", "qubits", "case", "seconds", "bytes_moved", "gate_count"], meta, args)
    return 0


def cmd_gate_bench(args) -> int:
    n = args.qubits
    sess = _session(args, n)
    m = n - sess.p
    ca = chunk_amps(args.chunk_bytes)
    check_memory(n, sess.p, sess.inproc, args.chunk_bytes or DEFAULT_CHUNK_BYTES)
    gate = random_unitary(np.random.default_rng(args.seed))
    if args.controlled_grid:
        if n < 2:
            raise ValueError("--controlled-grid needs at least 2 qubits")
        pairs = [(c, t) for c in range(n) for t in range(n) if c != t]
    else:
        lo, hi = parse_range(args.qubit_range or f"0:{n - 1}", 0, n - 1, "--qubit-range")
        pairs = [(None, k) for k in range(lo, hi + 1)]
    sess.start()
    try:
        states = sess.states(n)
        secs = []
        for c, t in pairs:
            one = Circuit(n, [GateOp(gate, t, control=c, name="U" if c is None else "CU")])
            secs.append(min(sess.timed(lambda: sess.run(states, one, None, ca)) for _ in range(max(1, args.reps))))
    finally:
        sess.close()
    if sess.rank != 0:
        return 0
    rows = []
    for (c, t), s in zip(pairs, secs):
        case = classify_case(t, c, m)
        moved = traffic_bytes(case, m)
        row = {"target": t, "case": case.case_id, "network": "yes" if case.case_id in (2, 5, 6) else "no",
               "seconds": f"{s:.6e}", "bytes_moved": moved, "gbps": f"{moved / s / 1e9:.3f}"}
        rows.append(row if c is None else {"control": c, **row})
    meta = {"command": "gate-bench", "n": n, "p": sess.p, "threads": args.threads, "grid": bool(args.controlled_grid),
            "seed": args.seed, "reps": args.reps}
    emit(rows, list(rows[0]), meta, args)
    return 0


def cmd_qft_bench(args) -> int:
    lo, hi = parse_range(args.qubits_range, 1, 64, "--qubits-range")
    sess = _session(args, lo)
    ca = chunk_amps(args.chunk_bytes)
    check_memory(hi, sess.p, sess.inproc, args.chunk_bytes or DEFAULT_CHUNK_BYTES)
    sizes = list(range(lo, hi + 1))
    sess.start()
    try:
        totals = []
        for n in sizes:
            circ = build_iqft(n) if args.inverse else build_qft(n)
            fusion = fusion_config(args.fusion, n - sess.p)
            states = sess.states(n)
            totals.append(sess.timed(lambda: sess.run(states, circ, fusion, ca)))
            del states
    finally:
        sess.close()
    if sess.rank != 0:
        return 0
    rows = [{"n": n, "ngates": n * (n + 1) // 2, "total_s": f"{t:.6e}", "s_per_gate": f"{t / (n * (n + 1) // 2):.6e}"}
            for n, t in zip(sizes, totals)]
    meta = {"command": "qft-bench", "p": sess.p, "threads": args.threads, "fusion": args.fusion or "off",
            "inverse": bool(args.inverse)}
    emit(rows, ["n", "ngates", "total_s", "s_per_gate"], meta, args)
    return 0


def probe_copy_bandwidth(nbytes: int = 4 << 30, reps: int = 5) -> float:
    """Device-to-device copy bandwidth (read + write bytes / s) of the current GPU."""
    import torch

    if not torch.cuda.is_available():
        raise ResourceError("--probe needs a CUDA device")
    a = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    b.copy_(a)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        b.copy_(a)
    e.record()
    e.synchronize()
    return 2 * nbytes * reps / (s.elapsed_time(e) * 1e-3)


def cmd_bounds(args) -> int:
    lo, hi = (args.m, args.m) if args.m is not None else parse_range(args.m_range, 1, 64, "--m-range")
    base = b200_params() if args.b200 else MachineParams()
    b_mem = probe_copy_bandwidth() if args.probe else (args.bmem if args.bmem is not None else base.b_mem)
    b_net = args.bnet if args.bnet is not None else base.b_net
    params = MachineParams(b_mem=b_mem, b_net=b_net, llc_bytes=base.llc_bytes)
    rows = [{"m": m, **{f"case{c.case_id}_s": f"{lower_bound_seconds(c, m, params):.4f}" for c in BoundCase}}
            for m in range(lo, hi + 1)]
    meta = {"command": "bounds", "b_mem": params.b_mem, "b_net": params.b_net,
            "machine": "b200" if args.b200 else "paper (Stampede socket)"}
    emit(rows, ["m"] + [f"case{c.case_id}_s" for c in BoundCase], meta, args)
    return 0


# ---------------------------------------------------------------- wiring


def _common(sub: argparse.ArgumentParser) -> None:
    sub.add_argument("--ranks", type=int, default=1, help="rank count, a power of two (torchrun: WORLD_SIZE)")
    sub.add_argument("--threads", type=int, default=1, help="accepted for compatibility; ignored on the GPU")
    sub.add_argument("--fusion", default=None, metavar="L_C|passes|off",
                     help="block exponent for gate fusion, 'passes' (native planner) or 'off' (default)")
    sub.add_argument("--chunk-bytes", type=int, default=None, help="exchange chunk size (validated; the fused "
                                                                   "NVLink kernel needs no staging)")
    sub.add_argument("--transport", default="inproc", help="inproc (default) or nvlink (torchrun)")
    sub.add_argument("--diagonal-local", action="store_true",
                     help="diagonal gates on global qubits without an exchange (torchrun runs)")
    sub.add_argument("--seed", type=int, default=0)
    sub.add_argument("--format", choices=("csv", "json"), default="csv")
    sub.add_argument("--out", default=None, help="output path (default stdout)")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1601_07195_b200",
                                 description="B200 state-vector simulator for gate circuits")
    subs = ap.add_subparsers(dest="command", required=True)
    run = subs.add_parser("run", help="execute a circuit file")
    run.add_argument("circuit")
    run.add_argument("--initial", type=int, default=0, help="initial basis index (default 0)")
    _common(run)
    gb = subs.add_parser("gate-bench", help="time single or controlled gates per position")
    gb.add_argument("--qubits", type=int, required=True)
    gb.add_argument("--qubit-range", default=None, help="lo:hi sweep range (default all)")
    gb.add_argument("--controlled-grid", action="store_true", help="every (control, target) pair")
    gb.add_argument("--reps", type=int, default=3, help="repetitions per point, best kept")
    _common(gb)
    qb = subs.add_parser("qft-bench", help="time transform circuits over a qubit range")
    qb.add_argument("--qubits-range", required=True, help="lo:hi inclusive")
    qb.add_argument("--inverse", action="store_true")
    _common(qb)
    bd = subs.add_parser("bounds", help="print the analytic lower-bound table")
    bd.add_argument("--m", type=int, default=None)
    bd.add_argument("--m-range", default="29:36")
    bd.add_argument("--b200", action="store_true",
                    help="B200 parameters (measured HBM copy peak, NVLink 5) instead of the paper's socket")
    bd.add_argument("--bmem", type=float, default=None, help="memory bytes/s (default 40e9, --b200: measured)")
    bd.add_argument("--bnet", type=float, default=None, help="network bytes/s, sent + received (default 5.5e9)")
    bd.add_argument("--probe", action="store_true", help="measure the GPU's copy bandwidth for --bmem")
    bd.add_argument("--format", choices=("csv", "json"), default="csv")
    bd.add_argument("--out", default=None)
    return ap


COMMANDS = {"run": cmd_run, "gate-bench": cmd_gate_bench, "qft-bench": cmd_qft_bench, "bounds": cmd_bounds}


def classify_failure(exc: BaseException) -> int:
    seen, cur = set(), exc
    while cur is not None and id(cur) not in seen:
        seen.add(id(cur))
        for cls, code in ((CircuitParseError, 3), (ResourceError, 4), (TransportError, 5)):
            if isinstance(cur, cls):
                return code
        if isinstance(cur, (LayoutError, FusionContractError, ValueError, OSError)):
            return 2
        cur = cur.__cause__
    return 1


def main(argv: list[str] | None = None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        return COMMANDS[args.command](args)
    except (OSError, RuntimeError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return classify_failure(exc)


if __name__ == "__main__":
    sys.exit(main())

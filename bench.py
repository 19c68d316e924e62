#!/usr/bin/env python
"""Benchmark of the gate-application hot path (BASELINE.json metric).

Default workload (N=1: BASELINE config 2): n = 30 + log2(N) qubits, 2^30
complex128 amplitudes (16 GiB) per GPU, seeded random normalised state; one
step = one per-target sweep, a fresh Haar-random 2x2 unitary on every qubit
k = 0..n-1 in order (at N > 1 the top log2(N) targets are global qubits and
run the fused NVLink exchange).  Weak scaling: per-GPU work is fixed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload sweep|controlled|random|qft] [--qubits N]

``--gpus N`` without torchrun launches N ranks itself (torch.distributed.run,
127.0.0.1); under torchrun WORLD_SIZE must equal N.  Prints ONE JSON line on
rank 0.  `value` is the effective HBM bandwidth per gate of the whole job,
(gates x 32 x 2^n bytes) / time (16 x 2^n for controlled gates), the paper's
"effective GB/s per gate"; `gates_per_s` rides along.
Timing: W untimed steps, then K steps between barrier+synchronize, CUDA
events on the launching stream, max over ranks.  The 16 GiB slice is ~130x
the 126 MB L2, so no flush is needed between steps.

The same line carries the BASELINE configs 3 / 4 / 5 shapes as secondary
objects (``secondary``: config-3 controlled gates per gate with (c, t) buckets
and through the pass planner, config-4-shaped random steps and the config-5
transform through the pass planner, exact and tolerance-mode), each with its
own roofline.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "gates/sec & effective HBM GB/s per gate vs 8 TB/s at n qubits; 1/2/4/8 GPU"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="GPUs (ranks) of the job; default WORLD_SIZE under torchrun, else 1")
    ap.add_argument("--steps", type=int, default=10, help="timed steps (BASELINE config 2: 10 repetitions of the sweep)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["sweep", "controlled", "random", "qft"], default="sweep")
    ap.add_argument("--qubits", dest="n", type=int, default=None, help="total qubits (default 30 + log2(N))")
    ap.add_argument("--fusion", choices=["none", "passes", "tolerance"], default=None,
                    help="none: one launch per gate (default, BASELINE config 2 is per-gate); "
                         "passes: native pass planner, bitwise (default for --workload qft); "
                         "tolerance: passes with exact=False (collapsed diagonals, 1e-12*sqrt(G) parity)")
    ap.add_argument("--l-c", type=int, default=12, help="register tile exponent for --fusion passes")
    ap.add_argument("--data-plane", choices=["ipc", "nccl", "ce"], default="ipc",
                    help="global-qubit exchanges: fused kernel on CUDA-IPC-mapped peer slices (default), the "
                         "reference's staged pipeline over NCCL send/recv (baseline) or copy-engine chunks")
    ap.add_argument("--diagonal-local", action="store_true",
                    help="diagonal gates on global qubits without an exchange (SURVEY.md 8(f)1; off by default: "
                         "it departs from the reference's per-gate NVLink traffic contract)")
    ap.add_argument("--remap", action="store_true",
                    help="global<->local qubit swaps instead of per-gate exchanges (SURVEY.md 8(f)4; N > 1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the config 3/4/5 secondary objects")
    ap.add_argument("--no-planes", action="store_true",
                    help="N > 1: skip timing one global-qubit gate on every exchange data plane (ipc, ce, nccl)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--out", default=None, help="also write the JSON line here")
    return ap.parse_args(argv)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def job_size(args, env=None) -> int:
    """Number of ranks of the job.  Under torchrun WORLD_SIZE decides and --gpus must agree;
    without it, --gpus (default 1)."""
    env = os.environ if env is None else env
    if "WORLD_SIZE" in env:
        world = int(env["WORLD_SIZE"])
        if args.gpus is not None and args.gpus != world:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                             f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus")
        n = world
    else:
        n = args.gpus or 1
    if n < 1 or n & (n - 1):
        raise SystemExit(f"bench.py: --gpus must be a power of two, got {n}")
    return n


def launch_command(args, argv, port: int) -> list[str] | None:
    """The torch.distributed.run command that fans --gpus N out to N ranks (one per GPU),
    or None when this process already is a rank / the job has one rank (the reference's
    run_spmd rank fan-out, pkg/src/svsim/transport.py:274-310)."""
    if "WORLD_SIZE" in os.environ or (args.gpus or 1) == 1:
        return None
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *argv]


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def step_circuits(sv, workload, n, count, seed=1):
    """One circuit per step (fresh Haar gates each step, same placement)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        if workload == "sweep":
            out.append(sv.per_target_sweep(n, 1, rng))
        elif workload == "controlled":  # BASELINE config 3 shape, 30 gates per step
            out.append(sv.random_circuit(n, 30, rng, controlled_fraction=1.0))
        elif workload == "random":  # BASELINE config 4 shape, 25 gates per step
            out.append(sv.random_circuit(n, 25, rng, controlled_fraction=0.0))
        else:
            out.append(sv.build_qft(n))
    return out


WORKLOADS = {
    "sweep": "BASELINE config 2: n={n}, one fresh Haar gate per target k=0..{n1} per step",
    "controlled": "BASELINE config 3 shape: n={n}, 30 Haar controlled gates per step, (c,t) uniform distinct",
    "random": "BASELINE config 4 shape: n={n}, 25 Haar single-qubit gates per step, targets uniform",
    "qft": "BASELINE config 5 shape: transform circuit build_qft(n={n}) per step",
}


def effective_bytes(circ, n):
    """Paper's effective bytes per gate: 32 x 2^n (16 x 2^n for controlled)."""
    return sum((32 if op.control is None else 16) << n for op in circ)


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clocks / throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], 0, False
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max, "reasons": names,
                "samples": len(self.samples)}


def load_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0}, "fallback"


def ncu_traffic(kernel_key, alg_bytes):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    (profiles/ncu_summary.json), rescaled to this launch's size when the capture used a smaller
    slice (traffic/algorithmic is size-independent once the slice is >> L2)."""
    try:
        d = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text())["kernels"][kernel_key]
        scale = alg_bytes / d.get("algorithmic_bytes", alg_bytes)
        out = {"dram_bytes_per_launch": round(d["dram_bytes_per_launch"] * scale),
               "captured_at_m": d.get("m"), "source": "profiles/ncu_summary.json"}
        return out["dram_bytes_per_launch"], out
    except (OSError, KeyError, ValueError, TypeError):
        return None, None


def cpu_baseline(sv, host_state, n, circ, seconds):
    """The oracle (C restatement of the reference's kernels, OpenMP) on the host copy of the state."""
    from oracle import oracle

    threads = os.cpu_count() or 1
    amps = host_state.numpy() if hasattr(host_state, "numpy") else host_state
    gates = 0
    nbytes = 0
    t0 = time.perf_counter()
    for op in circ:
        oracle.apply_gate(amps, op, threads=threads)
        gates += 1
        nbytes += (32 if op.control is None else 16) << n
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": round(nbytes / dt / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "gates_per_s": round(gates / dt, 4),
            "sample": f"first {gates} gates (targets {circ.gates[0].target}..{circ.gates[gates - 1].target}) "
                      f"of one n={n} step on the host copy of the state, oracle/sv_oracle.c with {threads} "
                      f"OpenMP threads, {dt:.2f} s"}


# ------------------------------------------------------------------ reference arm


def rank_share(oracle, amps, partner, op, m, rep_rank, threads):
    """One representative rank's share of one gate on the CPU port (oracle/sv_oracle.c):
    local gates on its 2^m slice, global targets as its half of the pairwise exchange
    against a second host slice standing in for the partner (distributed.py:187-422)."""
    t, c = op.target, op.control
    if t < m and (c is None or c < m):
        oracle.apply_gate(amps, op, threads=threads)
        return
    if t < m:  # control on a rank bit: the representative rank has it set
        oracle.apply_single(amps, t, op.gate, threads=threads)
        return
    own_zero = ((rep_rank >> (t - m)) & 1) == 0
    oracle.exchange(amps, partner, own_zero, -1 if c is None or c >= m else c, op.gate, threads=threads)


def stock_reference(n, circ, seconds):
    """The stock reference (baseline/_ref: svsim installed unmodified from /root/reference) through
    its public API, svsim.run_circuit(..., policy=ThreadPolicy(os.cpu_count())), on a bounded
    sample of the step's gates on a 2^n host state (engine.py:30-96, kernels.py:83-105)."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "svsim").exists():
        return {"unavailable": "baseline/_ref/svsim not installed"}
    sys.path.insert(0, str(ref))
    try:
        import svsim
        from svsim.kernels import ThreadPolicy
    except Exception as exc:  # noqa: BLE001
        return {"unavailable": f"import svsim failed: {exc!r}"}
    finally:
        sys.path.remove(str(ref))
    threads = os.cpu_count() or 1
    from oracle import oracle

    amps = np.empty(1 << n, dtype=np.complex128)
    oracle.fill_philox(amps, 0, 0, threads)
    state = svsim.LocalState(svsim.Layout(n, 0, 0), amps)
    policy = ThreadPolicy(threads)
    done, nbytes, t_all = 0, 0, 0.0
    for op in circ:
        one = svsim.Circuit(n, [svsim.GateOp(svsim.GateMatrix(op.gate.mat), op.target, op.control)])
        t0 = time.perf_counter()
        svsim.run_circuit(state, one, policy=policy)
        t_all += time.perf_counter() - t0
        done += 1
        nbytes += (32 if op.control is None else 16) << n
        if t_all > seconds:
            break
    return {"value": round(nbytes / t_all / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
            "gates": done, "seconds": round(t_all, 3),
            "sample": f"first {done} gates of the step, svsim.run_circuit(policy=ThreadPolicy({threads})) "
                      f"from baseline/_ref on a 2^{n} host state"}


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU algorithm on our config, rank 0 only.

    Timed: the oracle port (oracle/sv_oracle.c, the reference's arithmetic restated in C,
    OpenMP on every host thread) running the GPU arm's step circuits (same seeds, same
    per-step gates) on the same seeded state recipe.  At N = 1 each timed step is the whole
    step circuit (same_config).  At N > 1 the whole 2^n state does not fit one host: each step
    times one representative rank's share (every rank bit set, so every control-set rank's
    work is done) on a 2^m slice plus a partner slice, and the whole job is N such shares
    run back to back on the one host (the CPU path is memory-bound).  The stock reference
    (svsim from baseline/_ref) is timed beside it on a bounded sample (``stock_reference``)."""
    if rank != 0:
        return
    import paper_1601_07195_b200 as sv  # circuits only (the reference's RNG order), no kernels
    from oracle import oracle

    g = world.bit_length() - 1
    n = args.n or (30 + g)
    m = n - g
    rep = world - 1
    threads = os.cpu_count() or 1
    amps = np.empty(1 << m, dtype=np.complex128)
    oracle.fill_philox(amps, 0, rep, threads)
    partner = None
    if g:
        partner = np.empty(1 << m, dtype=np.complex128)
        oracle.fill_philox(partner, 0, rep ^ 1, threads)
    circs = step_circuits(sv, args.workload, n, args.warmup + args.steps)
    times, eff = [], 0
    for s, circ in enumerate(circs):
        ops = circ.gates if s >= args.warmup else circ.gates[:1]  # warm-up: page in, spin up threads
        t0 = time.perf_counter()
        for op in ops:
            rank_share(oracle, amps, partner, op, m, rep, threads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt * world)
            eff += effective_bytes(circ, n)
    tot = sum(times)
    value = eff / tot / 1e9
    stock = stock_reference(min(n, 30), circs[-1].gates if args.workload != "qft" else circs[-1].gates[:3],
                            args.cpu_seconds) if not args.no_cpu_baseline else None
    sample = (f"every gate of each of the {args.steps} step circuits on the seeded 2^{n} state" if g == 0 else
              f"rank {rep}'s share of every gate of each of the {args.steps} step circuits on a 2^{m} slice "
              f"(+ a partner slice for exchanges), x {world} ranks back to back on this host")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "gates_per_s": round(sum(len(c) for c in circs[args.warmup:]) / tot, 4),
        "config": {"workload": WORKLOADS[args.workload].format(n=n, n1=n - 1), "n_qubits": n, "local_qubits": m,
                   "global_qubits": g, "gates_per_step": len(circs[-1]), "seed": {"state": 0, "circuit": 1},
                   "same_config": g == 0, "sample": sample},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"{sample}; oracle/sv_oracle.c (C restatement of kernels.py:120-196, "
                                   f"distributed.py:187-202), {threads} OpenMP threads"},
        "stock_reference": stock,
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(line) + "\n")


# ------------------------------------------------------------------ GPU arm

# FP64 pipe ops per pair of the cheapest exact update each gate shape admits (svb200.cu spec_pair):
# general mix() 20, real 12, Hadamard-like 8, diagonal 8, phase 4 (one cmul on the |1> side).
FP64_OPS = {"general": 20, "real": 12, "hshare": 8, "diag": 8, "phase": 4}
FP64_PEAK_OPS = 17.0e12  # measured DFMA/DMUL issue rate, tools/micro/fp64_probe.cu


def gate_shape(q) -> str:
    q = np.asarray(q, dtype=np.complex128).reshape(2, 2)
    if q[0, 1] == 0 and q[1, 0] == 0:
        return "phase" if q[0, 0] == 1 else "diag"
    if np.all(q.imag == 0):
        return "hshare" if q[0, 0] == q[0, 1] == q[1, 0] == -q[1, 1] else "real"
    return "general"


def fp64_ops(gates, m) -> int:
    """Algorithmic FP64 ops of a gate list on a 2^m slice (local gates; controls halve the pairs)."""
    tot = 0
    for op in gates:
        pairs = 1 << (m - 1 - (op.control is not None))
        tot += FP64_OPS[gate_shape(op.gate.mat if hasattr(op.gate, "mat") else op.gate)] * pairs
    return tot


def p2p_probe(state, fabric, dev, barrier, reduce_scalar, nbytes=1 << 31, reps=3):
    """Measured NVLink denominator for the exchange kernels: every rank copies nbytes of its
    partner's (rank ^ 1) mapped slice into local memory with the copy engine (cudaMemcpyAsync
    on a CUDA-IPC peer pointer), all pairs at once, so each GPU sends and receives nbytes per
    copy -- the exchange's bidirectional load.  GB/s per direction, max-over-ranks time."""
    import torch
    import torch.distributed as dist

    fabric.ensure_registered(state)
    if fabric.data_plane == "nccl":
        return None
    nbytes = min(nbytes, 16 << state.layout.m)
    src = fabric.peer_pointer(state, fabric.rank ^ 1)
    buf = torch.empty(nbytes // 16, dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream()
    fabric.executor.copy(buf.data_ptr(), src, nbytes, state)  # warm-up (maps, TLBs)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fabric.executor.copy(buf.data_ptr(), src, nbytes, state)
    e1.record(stream)
    barrier()
    ms = reduce_scalar(e0.elapsed_time(e1), dist.ReduceOp.MAX)
    del buf
    return {"gbs_per_direction": round(reps * nbytes / (ms * 1e-3) / 1e9, 1), "bytes": nbytes, "reps": reps,
            "how": "cudaMemcpyAsync of the partner's (rank^1) CUDA-IPC-mapped slice, every rank at once"}


def make_units(sv, circ, m, fusion, l_c, state, fabric, remap=False):
    """The launch groups of one step: (kind, bytes, gate count, callable, gates); bytes are
    algorithmic HBM bytes for local units and NVLink bytes per direction for link units.

    Unfused: one unit per gate (the reference's engine.py:88-95 loop).  Passes:
    one unit per HBM pass of the native planner (passes.py).  remap: global<->local
    swaps (remap.py) instead of exchanges, the gates in between as above."""
    if remap and fabric is not None:
        items, _ = sv.plan_remapped(circ.gates, circ.n, m)
        units = []
        for it in items:
            if isinstance(it, sv.Swap):
                units.append(("swap", 1 << (m + 3), 0, (lambda it=it: sv.swap_global(state, it, fabric)), ()))
            else:
                units += make_units(sv, sv.Circuit(circ.n, it), m, fusion, l_c, state, fabric)
        return units
    if fusion in ("passes", "tolerance"):
        from paper_1601_07195_b200.passes import tile_for

        tile = tile_for(l_c, m)
        exact = fusion == "passes"
        return [("pass-" + p.kind + ("_tol" if not p.exact and p.kind == "local_stage" else ""),
                 (32 << m) if p.local else (1 << (m + 4)), len(p.gates),
                 (lambda p=p: sv.execute_pass(state, p, fabric, tile=tile)), p.gates)
                for p in sv.plan_passes(circ.gates, m, tile, exact=exact)]
    units = []
    for op in circ:
        case = sv.classify_case(op.target, op.control, m)
        if case in (sv.BoundCase.SINGLE_LOCAL, sv.BoundCase.CONTROLLED_REMOTE_CONTROL):
            kind, nbytes = "single", 32 << m
        elif case is sv.BoundCase.CONTROLLED_LOCAL:
            kind, nbytes = "controlled", 16 << m
        elif fabric is not None and fabric.diag_mode and sv.is_diagonal(op.gate):
            kind, nbytes = "diag-global", 32 << m  # sv_diag_global: one local pass, no exchange
        else:
            kind, nbytes = "exchange", sv.link_bytes_per_direction(case, m)
        units.append((kind, nbytes, 1, (lambda op=op: sv.apply_op(state, op, fabric)), (op,)))
    return units


KERNELS = {
    "single": ("sv_apply_single", "k_pairs/k_shfl<MODE_SINGLE> (sv_apply_single)"),
    "controlled": ("sv_apply_controlled", "k_pairs/k_shfl<MODE_CTL|MODE_PRED> (sv_apply_controlled)"),
    "pass-local_stage": ("sv_apply_gates:stage", "k_mstage (sv_apply_gates, multi-target stage pass; compiled control "
                                                 "flow for transform-shaped groups)"),
    "pass-local_tile": ("sv_apply_gates:tile", "k_tile (sv_apply_gates, register-tiled run)"),
    "pass-local_gate": ("sv_apply_single", "k_pairs/k_shfl (single gate of a pass plan)"),
    "pass-local_stage2": ("sv_apply_gates:dstage2", "k_xstage2 / k_dstage2 (tolerance mode: eight stage targets per "
                                                     "pass, two phases around a shared-memory transpose; compiled "
                                                     "phases for transform-shaped groups, the op interpreter otherwise)"),
    "pass-local_low": ("sv_apply_gates:low", "k_dlow (gates on qubits 0..5, one warp per 256 amplitudes; exact: "
                                            "speculative updates + zero test + replay; tolerance: diagonal runs as "
                                            "per-stage factors / 64-entry product tables)"),
    "pass-local_stage_tol": ("sv_apply_gates:dstage", "k_dstage (tolerance mode: diagonal runs folded into "
                                                      "per-byte product tables, k_dtable)"),
}
GLOBAL_KINDS = ("exchange", "swap", "pass-global_stage", "pass-global_gate")


class Timer:
    """Runs step circuits unit by unit with CUDA events on the launching stream."""

    def __init__(self, sv, torch, dist, world, stream, barrier, reduce_scalar, local):
        self.sv, self.torch, self.dist, self.world = sv, torch, dist, world
        self.stream, self.barrier, self.reduce_scalar, self.local = stream, barrier, reduce_scalar, local

    def run(self, circs, state, m, fabric, fusion, l_c, remap=False):
        torch, sv = self.torch, self.sv
        units = [make_units(sv, c, m, fusion, l_c, state, fabric, remap) for c in circs]
        ev = []
        launches0 = sv.launch_count()
        with ClockSampler(self.local) as clocks:
            self.barrier()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(self.stream)
            for us in units:
                row = [torch.cuda.Event(enable_timing=True)]
                row[0].record(self.stream)
                for _, _, _, fn, _ in us:
                    fn()
                    e = torch.cuda.Event(enable_timing=True)
                    e.record(self.stream)
                    row.append(e)
                ev.append(row)
            t1.record(self.stream)
            torch.cuda.synchronize()
        launches = sv.launch_count() - launches0
        elapsed = t0.elapsed_time(t1)
        if self.world > 1:
            elapsed = self.reduce_scalar(elapsed, self.dist.ReduceOp.MAX)
            launches = int(self.reduce_scalar(float(launches), self.dist.ReduceOp.SUM))
        unit_ms = [[row[i].elapsed_time(row[i + 1]) for i in range(len(row) - 1)] for row in ev]
        return {"elapsed_ms": elapsed, "unit_ms": unit_ms, "units": units, "launches": launches,
                "clocks": clocks.summary()}


def roofline(res, m, peaks, peak_kind):
    """Roofline of the dominant local kernel (largest share of the timed region)."""
    by_kind: dict = {}
    for us, ms in zip(res["units"], res["unit_ms"]):
        for (kind, nbytes, cnt, _, gates), t_ms in zip(us, ms):
            by_kind.setdefault(kind, []).append((nbytes, t_ms, cnt, gates))
    local_kinds = [k for k in by_kind if k in KERNELS]
    if not local_kinds:
        return None, by_kind
    top = max(local_kinds, key=lambda k: sum(r[1] for r in by_kind[k]))
    rows = by_kind[top]
    avg_ms = float(np.mean([r[1] for r in rows]))
    alg = int(np.mean([r[0] for r in rows]))
    achieved = alg / (avg_ms * 1e-3) / 1e9
    key, kname = KERNELS[top]
    traffic, tsrc = ncu_traffic(key, alg)
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": traffic, "traffic_source": tsrc,
            "kernel": kname, "peak_kind": peak_kind, "algorithmic_bytes_per_launch": alg,
            "avg_launch_ms": round(avg_ms, 4), "launches": len(rows),
            "share_of_step": round(sum(r[1] for r in rows) / res["elapsed_ms"], 4),
            "frac_of_8TBs": round(achieved / 8000.0, 4)}
    if top.startswith("pass-"):
        roof["gates_per_launch"] = round(float(np.mean([r[2] for r in rows])), 2)
        # fused passes are FP64-pipe bound once a pass carries enough gates: report that roofline too
        # (not for the tolerance-mode stage / low-bit kernels: they collapse diagonal runs, so the
        # per-gate op count of the exact updates is not what they execute)
        if top not in ("pass-local_stage2", "pass-local_low", "pass-local_stage_tol"):
            ops = float(np.mean([fp64_ops(r[3], m) for r in rows]))
            roof["fp64"] = {"achieved_tops": round(ops / (avg_ms * 1e-3) / 1e12, 3),
                            "peak_tops": FP64_PEAK_OPS / 1e12,
                            "frac": round(ops / (avg_ms * 1e-3) / FP64_PEAK_OPS, 4),
                            "ops_per_launch": int(ops), "peak_kind": "measured (tools/micro/fp64_probe.cu)",
                            "note": "op counts of the exact updates of the pass's gates"}
    return roof, by_kind


def controlled_buckets(circs, unit_ms, m):
    """GB/s (16*2^m accounting) by c<t / c>t and by min(c,t) / c."""
    buckets = {}
    for c_circ, ms in zip(circs, unit_ms):
        for op, t_ms in zip(c_circ, ms):
            if op.control is None or op.max_qubit() >= m:
                continue
            lo = min(op.control, op.target)
            band = "0" if lo == 0 else "1" if lo == 1 else "2-4" if lo <= 4 else ">=5"
            cb = str(op.control) if op.control <= 2 else ">=3"
            for key in (f"c<t" if op.control < op.target else "c>t", f"min(c,t)={band}", f"c={cb}"):
                buckets.setdefault(key, []).append(t_ms)
    return {k: {"gbps": round((16 << m) / (float(np.median(v)) * 1e-3) / 1e9, 1), "gates": len(v)}
            for k, v in sorted(buckets.items())}


def probe_and_exit(world, rank, n, m):
    """SVB_BENCH_PROBE=1: report the rank layout the launcher produced, then stop (CPU tests)."""
    print(json.dumps({"probe": True, "rank": rank, "world": world, "n_qubits": n, "local_qubits": m,
                      "global_qubits": n - m}), flush=True)


def run_ours(args, world, rank, local):
    import torch
    import torch.distributed as dist

    g = world.bit_length() - 1
    n = args.n or (30 + g)
    if os.environ.get("SVB_BENCH_PROBE") == "1":
        if world > 1:
            dist.init_process_group("gloo")
            dist.barrier()
        probe_and_exit(world, rank, n, n - g)
        if world > 1:
            dist.destroy_process_group()
        return

    import paper_1601_07195_b200 as sv

    # SVB_SHARE_DEVICE=1 (diagnostics only): every rank on cuda:0 over gloo with host fences,
    # to exercise the multi-rank bench path on a one-GPU box.  Never used for reported numbers.
    shared = os.environ.get("SVB_SHARE_DEVICE") == "1"
    if shared:
        local = 0
    elif world > torch.cuda.device_count():
        raise SystemExit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    fabric = None
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        fabric = sv.NvlinkFabric(data_plane=args.data_plane, diagonal_local=args.diagonal_local)
    lay = sv.Layout(n, g, rank)
    m = lay.m
    fusion = args.fusion or ("passes" if args.workload == "qft" else "none")
    circs = step_circuits(sv, args.workload, n, args.warmup + args.steps)
    state = sv.init_random_state(lay, seed=0, transport=fabric, device=dev)
    # full-size self-check: keep the initial slice, undo every step at the end
    free_b, _ = torch.cuda.mem_get_info(dev)
    initial = state.amps.clone() if free_b > 5 * (16 << lay.m) else None
    stream = torch.cuda.current_stream()
    applied = []  # (circuit, FusionConfig) in order, for the self-check

    def fcfg_of(f):
        if f == "passes":
            return sv.FusionConfig(l_c=args.l_c, passes=True)
        if f == "tolerance":
            return sv.FusionConfig(l_c=args.l_c, passes=True, exact=False)
        return None

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def reduce_scalar(x, op):
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(t, op=op)
        return float(t[0])

    timer = Timer(sv, torch, dist, world, stream, barrier, reduce_scalar, local)
    peaks, peak_kind = load_peaks()

    # ---------------------------------------------------------- warm-up
    for c in circs[: args.warmup]:
        for _, _, _, fn, _ in make_units(sv, c, m, fusion, args.l_c, state, fabric, args.remap):
            fn()
        applied.append((c, fcfg_of(fusion)))
    barrier()

    # ------------------------- NVLink reference: copy-engine peer read, all pairs at once
    p2p = p2p_probe(state, fabric, dev, barrier, reduce_scalar) if world > 1 else None

    # ------------------------------------------------ timed (device-resident)
    timed = circs[args.warmup:]
    res = timer.run(timed, state, m, fabric, fusion, args.l_c, args.remap)
    applied += [(c, fcfg_of(fusion)) for c in timed]
    elapsed_ms = res["elapsed_ms"]
    ngates = sum(len(c) for c in timed)
    eff = sum(effective_bytes(c, n) for c in timed)
    value = eff / (elapsed_ms * 1e-3) / 1e9
    roof, by_kind = roofline(res, m, peaks, peak_kind)
    per_target = {}
    if args.workload == "sweep" and fusion == "none":
        for k in range(m):
            ks = [res["unit_ms"][j][k] for j in range(len(timed))]
            per_target[k] = round((32 << m) / (float(np.median(ks)) * 1e-3) / 1e9, 1)
    buckets = controlled_buckets(timed, res["unit_ms"], m) if args.workload == "controlled" and fusion == "none" \
        else {}
    nvlink = nvlink_summary(by_kind, world, p2p, len(timed))

    # ------------------------ secondary objects: BASELINE configs 3 / 4 / 5 shapes, same slice
    secondary = {}
    if not args.no_secondary and args.n is None:
        plan = [("controlled", "controlled", "none"), ("controlled_passes", "controlled", "passes"),
                ("random_passes", "random", "passes"),
                ("random_tolerance", "random", "tolerance"),
                ("qft_passes", "qft", "passes"), ("qft_tolerance", "qft", "tolerance")]
        for name, wl, fz in plan:
            if wl == args.workload and fz == fusion:
                continue
            sc = step_circuits(sv, wl, n, args.warmup + args.steps, seed=1)
            for c in sc[: args.warmup]:
                for _, _, _, fn, _ in make_units(sv, c, m, fz, args.l_c, state, fabric):
                    fn()
            barrier()
            r2 = timer.run(sc[args.warmup:], state, m, fabric, fz, args.l_c)
            applied += [(c, fcfg_of(fz)) for c in sc]
            rf, bk = roofline(r2, m, peaks, peak_kind)
            ms = r2["elapsed_ms"]
            obj = {"workload": WORKLOADS[wl].format(n=n, n1=n - 1),
                   "fusion": fz if fz == "none" else f"{fz} (l_c={args.l_c})",
                   "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
                   "value": round(sum(effective_bytes(c, n) for c in sc[args.warmup:]) / (ms * 1e-3) / 1e9, 3),
                   "unit": "GB/s", "gates_per_step": len(sc[-1]),
                   "gates_per_s": round(sum(len(c) for c in sc[args.warmup:]) / (ms * 1e-3), 3),
                   "hbm_passes_per_step": round(sum(len(u) for u in r2["units"]) / len(r2["units"]), 2),
                   "roofline": rf, "gpu_launches": r2["launches"], "clocks": r2["clocks"]}
            if wl == "controlled" and fz == "none":
                obj["buckets"] = controlled_buckets(sc[args.warmup:], r2["unit_ms"], m)
            nv2 = nvlink_summary(bk, world, p2p, args.steps)
            if nv2:
                obj["nvlink"] = nv2
            secondary[name] = obj

    # ------------------------------ N > 1: every exchange data plane on the same box
    planes = None
    if not args.no_planes and world > 1 and fabric is not None and fabric.data_plane != "nccl":
        planes = time_planes(sv, torch, dist, state, fabric, n, m, timer, args, p2p)

    # ------------------------------ self-check: inverse circuits restore the input
    self_check = None
    if initial is not None:
        tol_gates = 0
        for c, fc in reversed(applied):
            sv.run_circuit(state, c.inverse(), fabric, fusion=fc)
            if fc is not None and not fc.exact:
                tol_gates += 2 * len(c)
        from paper_1601_07195_b200.core import max_abs_diff

        err = max_abs_diff(state.amps, initial)
        if world > 1:
            err = reduce_scalar(err, dist.ReduceOp.MAX)
        ng = 2 * sum(len(c) for c, _ in applied)
        self_check = {"max_abs_err": err, "bound": 1e-12 * ng ** 0.5, "gates": ng,
                      "ok": err <= 1e-12 * ng ** 0.5,
                      "what": "every warm-up and timed step (main and secondary) undone by its inverse circuit, "
                              "vs the saved input"}
        if tol_gates:
            self_check["tolerance_mode_gates"] = tol_gates
        del initial

    # ---------------------------------------------- end to end (host buffers)
    e2e = None
    cpu = None
    import psutil

    fcfg = fcfg_of(fusion)
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    host_fits = (16 << m) * local_world <= 0.6 * psutil.virtual_memory().total
    if not args.no_e2e and not host_fits:  # decided alike on every rank: no collective diverges
        e2e = {"value": None, "unit": "GB/s", "skipped": f"one pinned {16 << m}-byte slice per rank x "
               f"{local_world} ranks exceeds 60% of this node's {psutil.virtual_memory().total} bytes of RAM"}
    if not args.no_e2e and host_fits:
        free_dev = torch.cuda.mem_get_info(dev)[0]
        # run_pipelined needs two or three device slots next to the state (three: upload i+1 runs
        # while download i-1 drains); otherwise the state itself is loaded and stored in turn
        pipelined = (2 * (16 << m) * local_world <= 0.45 * psutil.virtual_memory().total
                     and free_dev > 2.2 * (16 << m))
        nslot = 3 if free_dev > 3.3 * (16 << m) else 2
        h_in = torch.empty(lay.local_len, dtype=torch.complex128, pin_memory=True)
        h_out = torch.empty(lay.local_len, dtype=torch.complex128, pin_memory=True) if pipelined else h_in
        state.store_host(h_in)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        # every step: pinned H2D of its input, the circuit, D2H of its result
        if pipelined:  # public run_pipelined overlaps step i+1's upload / step i-1's download with step i
            sv.run_pipelined(lay, timed, [h_in] * len(timed), [h_out] * len(timed), fabric, fusion=fcfg,
                             slots=nslot)
        else:  # one host buffer per rank: sequential upload -> gates -> download
            for c in timed:
                state.load_host(h_in)
                sv.run_circuit(state, c, fabric, fusion=fcfg)
                state.store_host(h_in)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1)
        if world > 1:
            e2e_ms = reduce_scalar(e2e_ms, dist.ReduceOp.MAX)
        e2e = {"value": round(eff / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": (16 << m) * world, "d2h_bytes_per_step": (16 << m) * world,
               "ms_per_step": round(e2e_ms / len(timed), 3),
               "path": ("run_pipelined: LocalState.load_host (sv_copy, H2D stream) -> run_circuit -> "
                        f"LocalState.store_host (sv_copy, D2H stream), {nslot} device slots") if pipelined else
                       "sequential LocalState.load_host -> run_circuit -> store_host (host RAM bound)"}
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(sv, h_in, n, timed[0], args.cpu_seconds)
        del h_in, h_out

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(elapsed_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "gates_per_s": round(ngates / (elapsed_ms * 1e-3), 3),
            "config": {"workload": WORKLOADS[args.workload].format(n=n, n1=n - 1),
                       "fusion": fusion if fusion == "none" else f"{fusion} (l_c={args.l_c})",
                       "n_qubits": n, "local_qubits": m, "global_qubits": g, "gates_per_step": len(timed[0]),
                       "state_gib_per_gpu": (16 << m) / 2**30, "parallelism": f"state sharded over {world} GPU(s)",
                       "data_plane": fabric.data_plane if fabric is not None else None,
                       "diagonal_local": bool(fabric is not None and fabric.diag_mode),
                       "remap": bool(args.remap and fabric is not None),
                       "l2": "no flush: slice >> 126 MB L2" if m >= 26 else "slice fits L2 (parity-size run)",
                       "seed": {"state": 0, "circuit": 1}},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": res["launches"],
            "self_check": self_check, "clocks": res["clocks"],
        }
        if buckets:
            line["controlled_buckets"] = buckets
        if per_target:
            line["per_target_gbps"] = per_target
        if nvlink:
            line["nvlink"] = nvlink
        if planes:
            line["planes"] = planes
        if secondary:
            line["secondary"] = secondary
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            Path(args.out).write_text(s + "\n")
    if fabric is not None:
        fabric.close()
        dist.destroy_process_group()


def nvlink_summary(by_kind, world, p2p, steps):
    glob = [r for k, rs in by_kind.items() if k in GLOBAL_KINDS for r in rs]
    if world <= 1 or not glob:
        return None
    d = float(np.mean([r[1] for r in glob]))
    ach = sum(r[0] for r in glob) / (sum(r[1] for r in glob) * 1e-3) / 1e9  # link bytes per direction / time
    return {"achieved_gbs_per_direction": round(ach, 1),
            "peak_nominal": 900.0, "peak_measured_p2p": p2p["gbs_per_direction"] if p2p else None,
            "frac_nominal": round(ach / 900.0, 4),
            "frac_measured": round(ach / p2p["gbs_per_direction"], 4) if p2p else None, "p2p_probe": p2p,
            "global_launches_per_step": len(glob) // max(1, steps), "avg_ms": round(d, 3)}


def time_planes(sv, torch, dist, state, fabric, n, m, timer, args, p2p):
    """One global-qubit gate (target n-1) through each exchange data plane, same box, same slice:
    the fused IPC kernel (product), copy-engine chunks, NCCL send/recv chunks (baseline)."""
    out = {}
    rng = np.random.default_rng(99)
    circs = [sv.Circuit(n, [sv.GateOp(sv.random_unitary(rng), n - 1)]) for _ in range(args.warmup + 3)]
    orig = fabric.data_plane
    for plane in ("ipc", "ce", "nccl"):
        fabric.data_plane = plane
        for c in circs[: args.warmup]:
            sv.run_circuit(state, c, fabric)
        r = timer.run(circs[args.warmup:], state, m, fabric, "none", args.l_c)
        ms = r["elapsed_ms"] / 3
        gbs = (1 << (m + 4)) / (ms * 1e-3) / 1e9
        out[plane] = {"ms_per_gate": round(ms, 3), "gbs_per_direction": round(gbs, 1),
                      "frac_nominal": round(gbs / 900.0, 4),
                      "frac_measured": round(gbs / p2p["gbs_per_direction"], 4) if p2p else None}
        for c in reversed(circs):  # restore the slice for the self-check
            sv.run_circuit(state, c.inverse(), fabric)
    fabric.data_plane = orig
    return out


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    world = job_size(args)
    _, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return 0
    cmd = launch_command(args, argv, free_port())
    if cmd is not None:  # fan out: one rank per GPU, rank 0 prints the line
        return subprocess.call(cmd, env={**os.environ, "PYTHONUNBUFFERED": "1"})
    run_ours(args, world, rank, local)
    return 0


if __name__ == "__main__":
    sys.exit(main())

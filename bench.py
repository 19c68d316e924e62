#!/usr/bin/env python
"""Benchmark of the gate-application hot path (BASELINE.json metric).

Default workload (N=1: BASELINE config 2): n = 30 + log2(N) qubits, 2^30
complex128 amplitudes (16 GiB) per GPU, seeded random normalised state; one
step = one per-target sweep, a fresh Haar-random 2x2 unitary on every qubit
k = 0..n-1 in order (at N > 1 the top log2(N) targets are global qubits and
run the fused NVLink exchange).  Weak scaling: per-GPU work is fixed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload sweep|controlled|random|qft] [--n N]

Prints ONE JSON line on rank 0.  `value` is the effective HBM bandwidth per
gate of the whole job, (gates x 32 x 2^n bytes) / time, the paper's
"effective GB/s per gate"; `gates_per_s` rides along.
Timing: W untimed steps, then K steps between barrier+synchronize, CUDA
events on the launching stream, max over ranks.  The 16 GiB slice is ~130x
the 126 MB L2, so no flush is needed between steps.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "gates/sec & effective HBM GB/s per gate vs 8 TB/s at n qubits; 1/2/4/8 GPU"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10, help="timed steps (BASELINE config 2: 10 repetitions of the sweep)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["sweep", "controlled", "random", "qft"], default="sweep")
    ap.add_argument("--qubits", dest="n", type=int, default=None, help="total qubits (default 30 + log2(N))")
    ap.add_argument("--fusion", choices=["none", "passes"], default=None,
                    help="none: one launch per gate (default, BASELINE config 2 is per-gate); "
                         "passes: native pass planner (default for --workload qft)")
    ap.add_argument("--l-c", type=int, default=12, help="register tile exponent for --fusion passes")
    ap.add_argument("--data-plane", choices=["ipc", "nccl"], default="ipc",
                    help="global-qubit exchanges: fused kernel on CUDA-IPC-mapped peer slices (default) or the "
                         "reference's staged pipeline over NCCL send/recv (baseline)")
    ap.add_argument("--diagonal-local", action="store_true",
                    help="diagonal gates on global qubits without an exchange (SURVEY.md 8(f)1; off by default: "
                         "it departs from the reference's per-gate NVLink traffic contract)")
    ap.add_argument("--remap", action="store_true",
                    help="global<->local qubit swaps instead of per-gate exchanges (SURVEY.md 8(f)4; N > 1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--out", default=None, help="also write the JSON line here")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


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
        return round(d["dram_bytes_per_launch"] * scale)
    except (OSError, KeyError, ValueError, TypeError):
        return None


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


def run_reference(args):
    """--impl reference: the reference's CPU algorithm (oracle port, all host threads) on our config."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import paper_1601_07195_b200 as sv
    from oracle import oracle

    g = world.bit_length() - 1
    n = args.n or (30 + g)
    m = n - g
    threads = os.cpu_count() or 1
    # One host holds one rank's 2^m slice (16 GiB at the default size): the CPU
    # path is memory-bound, so the whole job on one host runs each gate's
    # per-rank shares back to back and whole-job GB/s equals the slice rate.
    amps = np.empty(1 << m, dtype=np.complex128)
    oracle.fill_phase(amps, threads)
    pool = [op for op in step_circuits(sv, args.workload, n, 1)[0].gates if op.max_qubit() < m]
    times, eff = [], 0
    for s in range(args.warmup + args.steps):
        op = pool[(s * 7) % len(pool)]
        t0 = time.perf_counter()
        oracle.apply_gate(amps, op, threads=threads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            eff += (32 if op.control is None else 16) << m
    tot = sum(times)
    value = eff / tot / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "gates_per_s": round(args.steps / tot, 4),
        "config": {"workload": WORKLOADS[args.workload].format(n=n, n1=n - 1), "n_qubits": n, "local_qubits": m,
                   "sample": f"one local gate of the step per timed step (target 7*s mod len), on one "
                             f"2^{m}-amplitude rank slice"},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} gates of the step on a 2^{m}-amplitude host slice, "
                                   f"oracle/sv_oracle.c (C restatement of kernels.py:120-196), {threads} threads"},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(line) + "\n")


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
    if fabric.data_plane != "ipc":
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
    if fusion == "passes":
        from paper_1601_07195_b200.passes import tile_for

        tile = tile_for(l_c, m)
        return [("pass-" + p.kind, (32 << m) if p.local else (1 << (m + 4)), len(p.gates),
                 (lambda p=p: sv.execute_pass(state, p, fabric, tile=tile)), p.gates)
                for p in sv.plan_passes(circ.gates, m, tile)]
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
    "pass-local_stage": ("sv_apply_gates:stage", "k_mstage (sv_apply_gates, multi-target stage pass)"),
    "pass-local_tile": ("sv_apply_gates:tile", "k_tile (sv_apply_gates, register-tiled run)"),
    "pass-local_gate": ("sv_apply_single", "k_pairs/k_shfl (single gate of a pass plan)"),
}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_1601_07195_b200 as sv

    world, rank, local = dist_env()
    # SVB_SHARE_DEVICE=1 (diagnostics only): every rank on cuda:0 over gloo with host fences,
    # to exercise the multi-rank bench path on a one-GPU box.  Never used for reported numbers.
    shared = os.environ.get("SVB_SHARE_DEVICE") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    fabric = None
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        fabric = sv.NvlinkFabric(data_plane=args.data_plane, diagonal_local=args.diagonal_local)
    if world & (world - 1):
        raise SystemExit("--gpus must be a power of two")
    g = world.bit_length() - 1
    n = args.n or (30 + g)
    lay = sv.Layout(n, g, rank)
    m = lay.m
    fusion = args.fusion or ("passes" if args.workload == "qft" else "none")
    circs = step_circuits(sv, args.workload, n, args.warmup + args.steps)
    state = sv.init_random_state(lay, seed=0, transport=fabric, device=dev)
    # full-size self-check: keep the initial slice, undo every step at the end
    free_b, _ = torch.cuda.mem_get_info(dev)
    initial = state.amps.clone() if free_b > 5 * (16 << lay.m) else None
    stream = torch.cuda.current_stream()
    fcfg = sv.FusionConfig(l_c=args.l_c, passes=True) if fusion == "passes" else None

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def reduce_scalar(x, op):
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(t, op=op)
        return float(t[0])

    # ---------------------------------------------------------- warm-up
    for c in circs[: args.warmup]:
        for _, _, _, fn, _ in make_units(sv, c, m, fusion, args.l_c, state, fabric, args.remap):
            fn()
    barrier()

    # ------------------------- NVLink reference: copy-engine peer read, all pairs at once
    p2p = p2p_probe(state, fabric, dev, barrier, reduce_scalar) if world > 1 else None

    # ------------------------------------------------ timed (device-resident)
    timed = circs[args.warmup:]
    units = [make_units(sv, c, m, fusion, args.l_c, state, fabric, args.remap) for c in timed]
    ev = []
    launches0 = sv.launch_count()
    with ClockSampler(local) as clocks:
        barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for us in units:
            row = [torch.cuda.Event(enable_timing=True)]
            row[0].record(stream)
            for _, _, _, fn, _ in us:
                fn()
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                row.append(e)
            ev.append(row)
        t_end.record(stream)
        torch.cuda.synchronize()
    launches = sv.launch_count() - launches0
    elapsed_ms = t_start.elapsed_time(t_end)
    if world > 1:
        elapsed_ms = reduce_scalar(elapsed_ms, dist.ReduceOp.MAX)
        launches = int(reduce_scalar(float(launches), dist.ReduceOp.SUM))
    unit_ms = [[row[i].elapsed_time(row[i + 1]) for i in range(len(row) - 1)] for row in ev]
    ngates = sum(len(c) for c in timed)
    eff = sum(effective_bytes(c, n) for c in timed)
    value = eff / (elapsed_ms * 1e-3) / 1e9

    # roofline of the dominant local kernel (largest share of the step)
    peaks, peak_kind = load_peaks()
    by_kind: dict = {}
    for us, ms in zip(units, unit_ms):
        for (kind, nbytes, cnt, _, gates), t_ms in zip(us, ms):
            by_kind.setdefault(kind, []).append((nbytes, t_ms, cnt, gates))
    local_kinds = [k for k in by_kind if k in KERNELS]
    roof = None
    if local_kinds:
        top = max(local_kinds, key=lambda k: sum(r[1] for r in by_kind[k]))
        rows = by_kind[top]
        avg_ms = float(np.mean([r[1] for r in rows]))
        alg = int(np.mean([r[0] for r in rows]))
        achieved = alg / (avg_ms * 1e-3) / 1e9
        key, kname = KERNELS[top]
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": ncu_traffic(key, alg),
                "kernel": kname, "peak_kind": peak_kind, "algorithmic_bytes_per_launch": alg,
                "avg_launch_ms": round(avg_ms, 4), "launches": len(rows),
                "share_of_step": round(sum(r[1] for r in rows) / elapsed_ms, 4),
                "frac_of_8TBs": round(achieved / 8000.0, 4)}
        if top.startswith("pass-"):
            roof["gates_per_launch"] = round(float(np.mean([r[2] for r in rows])), 2)
            # fused passes are FP64-pipe bound once a pass carries enough gates: report that roofline too
            ops = float(np.mean([fp64_ops(r[3], m) for r in rows]))
            roof["fp64"] = {"achieved_tops": round(ops / (avg_ms * 1e-3) / 1e12, 3),
                            "peak_tops": FP64_PEAK_OPS / 1e12, "frac": round(ops / (avg_ms * 1e-3) / FP64_PEAK_OPS, 4),
                            "ops_per_launch": int(ops), "peak_kind": "measured (tools/micro/fp64_probe.cu)"}
    per_target = {}
    if args.workload == "sweep" and fusion == "none":
        for k in range(m):
            ks = [unit_ms[j][k] for j in range(len(timed))]
            per_target[k] = round((32 << m) / (float(np.median(ks)) * 1e-3) / 1e9, 1)
    buckets = {}
    if args.workload == "controlled" and fusion == "none":
        # GB/s (16*2^m accounting) by c<t / c>t and by min(c,t)
        for c_circ, ms in zip(timed, unit_ms):
            for op, t_ms in zip(c_circ, ms):
                if op.control is None or op.max_qubit() >= m:
                    continue
                lo = min(op.control, op.target)
                band = "0" if lo == 0 else "1" if lo == 1 else "2-4" if lo <= 4 else ">=5"
                for key in (f"c<t" if op.control < op.target else "c>t", f"min(c,t)={band}"):
                    buckets.setdefault(key, []).append(t_ms)
        buckets = {k: {"gbps": round((16 << m) / (float(np.median(v)) * 1e-3) / 1e9, 1), "gates": len(v)}
                   for k, v in sorted(buckets.items())}
    nvlink = None
    glob = [r for k, rs in by_kind.items() if k in ("exchange", "swap", "pass-global_stage", "pass-global_gate")
            for r in rs]
    if world > 1 and glob:
        d = float(np.mean([r[1] for r in glob]))
        ach = sum(r[0] for r in glob) / (sum(r[1] for r in glob) * 1e-3) / 1e9  # link bytes per direction / time
        nvlink = {"achieved_gbs_per_direction": round(ach, 1),
                  "peak_nominal": 900.0, "peak_measured_p2p": p2p["gbs_per_direction"] if p2p else None,
                  "frac_nominal": round(ach / 900.0, 4),
                  "frac_measured": round(ach / p2p["gbs_per_direction"], 4) if p2p else None, "p2p_probe": p2p,
                  "global_launches_per_step": len(glob) // len(timed), "avg_ms": round(d, 3)}

    # ------------------------------ self-check: inverse circuits restore the input
    self_check = None
    if initial is not None:
        for c in reversed(circs):
            sv.run_circuit(state, c.inverse(), fabric, fusion=fcfg)
        from paper_1601_07195_b200.core import max_abs_diff

        err = max_abs_diff(state.amps, initial)
        if world > 1:
            err = reduce_scalar(err, dist.ReduceOp.MAX)
        ng = 2 * sum(len(c) for c in circs)
        self_check = {"max_abs_err": err, "bound": 1e-12 * ng ** 0.5, "gates": ng,
                      "ok": err <= 1e-12 * ng ** 0.5,
                      "what": "every warm-up and timed step undone by its inverse circuit, vs the saved input"}
        del initial

    # ---------------------------------------------- end to end (host buffers)
    e2e = None
    cpu = None
    import psutil

    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    host_fits = (16 << m) * local_world <= 0.6 * psutil.virtual_memory().total
    if not args.no_e2e and not host_fits:  # decided alike on every rank: no collective diverges
        e2e = {"value": None, "unit": "GB/s", "skipped": f"one pinned {16 << m}-byte slice per rank x "
               f"{local_world} ranks exceeds 60% of this node's {psutil.virtual_memory().total} bytes of RAM"}
    if not args.no_e2e and host_fits:
        # pinned host buffers for every rank on this node must fit comfortably in RAM
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
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "self_check": self_check,
            "clocks": clocks.summary(),
        }
        if buckets:
            line["controlled_buckets"] = buckets
        if per_target:
            line["per_target_gbps"] = per_target
        if nvlink:
            line["nvlink"] = nvlink
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            Path(args.out).write_text(s + "\n")
    if fabric is not None:
        fabric.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Summarise ncu captures into profiles/ (run here, on the CPU box, after a gpurun profiling call).

    python profiles/summarize_ncu.py --round r01 --launches gpurun_out/launches.csv \
        --rep sv_apply_single=gpurun_out/prof_pairs.ncu-rep [--rep key=path ...]

Writes profiles/<round>_launches.md (per-kernel share of the step from the
launch list) and merges per-launch DRAM traffic of each --rep into
profiles/ncu_summary.json, which bench.py reads for roofline.traffic.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict
from pathlib import Path

HERE = Path(__file__).resolve().parent
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
    "launch__occupancy_limit_registers", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1, "second": 1}


def raw_metrics(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                d[m] = v * SCALE.get(units[i], 1)
                d[m + ".unit"] = units[i]
        stalls = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: float(vals[i].replace(",", "") or 0)
                  for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")}
        tot = sum(stalls.values())
        if tot:
            d["stalls"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]}
        res.append(d)
    return res


def launches(path: str) -> str:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = ["| kernel | launches | total ms | share | avg us |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / 1e6:.3f} | {sum(v) / tot:.3f} | {sum(v) / len(v) / 1e3:.1f} |")
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--note", default="")
    ap.add_argument("--out", default=None, help="markdown name (default <round>_ncu.md)")
    ap.add_argument("--alg-bytes", type=float, default=None, help="algorithmic bytes per launch of the captures")
    a = ap.parse_args()
    md = [f"# ncu summary {a.round}", "", a.note, ""]
    if a.launches:
        md += ["## Launch list (cold-cache, serialised: compare shares)", "", launches(a.launches), ""]
    summ_path = HERE / "ncu_summary.json"
    summ = json.loads(summ_path.read_text()) if summ_path.exists() else {"kernels": {}}
    for spec in a.rep:
        key, rep = spec.split("=", 1)
        for i, d in enumerate(raw_metrics(rep)):
            rd, wr = d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)
            t = d.get("gpu__time_duration.sum", 0)
            md += [f"## `{key}` launch {i}: `{d['kernel'][:100]}`", "",
                   "| metric | value |", "|---|---|"]
            for m in METRICS:
                if m in d:
                    md.append(f"| {m} | {d[m]:.6g} |")
            if "stalls" in d:
                md.append("| top warp stall reasons (share of PC samples) | " +
                          ", ".join(f"{k} {v:.2f}" for k, v in d["stalls"].items()) + " |")
            md += [f"| dram bytes (read+write) | {rd + wr:.6g} |",
                   f"| dram GB/s (ncu, serialised replay) | {(rd + wr) / t / 1e9 if t else 0:.1f} |", ""]
            if i == 0:
                summ["kernels"][key] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                                        "duration_s": t, "kernel": d["kernel"], "round": a.round,
                                        "registers": d.get("launch__registers_per_thread"),
                                        "dram_pct_peak": d.get(
                                            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")}
                if a.alg_bytes:
                    summ["kernels"][key]["algorithmic_bytes"] = int(a.alg_bytes)
    (HERE / (a.out or f"{a.round}_ncu.md")).write_text("\n".join(md) + "\n")
    summ_path.write_text(json.dumps(summ, indent=1) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()

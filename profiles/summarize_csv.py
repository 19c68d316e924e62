"""Markdown summary of one `ncu --set full --import-source on` capture from its CSV exports
(the .ncu-rep files of the fused kernels are 35 MB each, over gpurun's copy-back limit, so
the GPU box exports them: `ncu -i rep --page raw --csv` and `--page source --csv --print-source sass`).

    python profiles/summarize_csv.py TITLE raw.csv sass.csv.gz >> profiles/rNN_ncu_xxx.md

Prints the headline metrics, the warp-stall shares, the issued-instruction mix by class, the
LDL/STL (spill) share of issued instructions and the ten hottest instructions by PC samples.
"""
import collections
import csv
import gzip
import re
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum", "smsp__inst_executed.sum",
]


def klass(src):
    t = src.split()
    op = t[0] if not t[0].startswith("@") else t[1]
    if re.match(r"D(FMA|MUL|ADD|SETP)", op):
        return "fp64"
    for pre, k in (("LDGSTS", "cp.async"), ("LDG", "ldg"), ("STG", "stg"), ("LDL", "local"), ("STL", "local"),
                   ("LDS", "smem"), ("STS", "smem"), ("LDC", "ldc"), ("BAR", "bar"), ("SHFL", "warp"), ("VOTE", "warp")):
        if op.startswith(pre):
            return k
    if op.startswith(("BRA", "BRX", "BSSY", "BSYNC", "EXIT", "CALL", "RET", "JMP", "WARPSYNC")):
        return "branch"
    return "uniform" if op.startswith("U") else "alu"


def main():
    title, raw, sass = sys.argv[1:4]
    rows = list(csv.reader(open(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    print(f"## {title}\n\n`{v[h.index('Kernel Name')]}`\n\n| metric | value |\n|---|---|")
    for w in WANT:
        if w in h:
            i = h.index(w)
            print(f"| {w} | {v[i]} {u[i]} |")
    rows = list(csv.reader(gzip.open(sass, "rt")))
    hdr, data = rows[1], rows[2:]
    ix = {c: i for i, c in enumerate(hdr)}
    tot = sum(int(r[ix["# Samples"]]) for r in data)
    stalls = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    agg = collections.Counter()
    for r in data:
        for s in stalls:
            agg[s] += int(r[ix[s]] or 0)
    print("| warp stall shares (PC samples) | " + ", ".join(f"{k[6:]} {x / tot:.2f}" for k, x in agg.most_common(8)) + " |")
    ex, sm = collections.Counter(), collections.Counter()
    for r in data:
        k = klass(r[ix["Source"]])
        ex[k] += int(r[ix["Instructions Executed"]])
        sm[k] += int(r[ix["# Samples"]])
    te = sum(ex.values())
    print("| issued warp instructions by class | " + ", ".join(f"{k} {x / te:.3f}" for k, x in ex.most_common()) + " |")
    print("| PC samples by class | " + ", ".join(f"{k} {x / tot:.3f}" for k, x in sm.most_common()) + " |")
    print(f"| SASS instructions / LDL+STL among them / LDL+STL share of issued | {len(data)} / "
          f"{sum(1 for r in data if klass(r[ix['Source']]) == 'local')} / {ex['local'] / te:.4f} |")
    print("\nHottest instructions (PC samples, executed warp instructions, top stall):\n\n```")
    for r in sorted(data, key=lambda r: -int(r[ix["# Samples"]]))[:10]:
        st = {s: int(r[ix[s]] or 0) for s in stalls}
        print(f"{r[ix['Source']].strip()[:64]:64s} {r[ix['# Samples']]:>7s} {r[ix['Instructions Executed']]:>10s} "
              f"{max(st, key=st.get)[6:]}")
    print("```\n")


main()

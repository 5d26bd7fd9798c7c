"""Summarise an ncu report (raw + source pages) as markdown for profiles/.

Usage: python tools/ncu_summary.py <report.ncu-rep> [title] > profiles/<name>.md
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    raw = ncu_csv(rep, "raw")
    hdr, units = raw[0], raw[1]
    print(f"# ncu summary: {title}\n")
    print(f"Source report: `{rep}` (ncu --set full --clock-control none --import-source on)\n")
    for row in raw[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print(f"## {d.get('Kernel Name', '?')}\n")
        print("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in d:
                print(f"| {label} (`{k}`) | {d[k]} {u.get(k, '')} |")
        stalls = sorted(((h, d[h]) for h in hdr
                         if h.startswith("smsp__average_warps_issue_stalled_")
                         and h.endswith("per_issue_active.ratio")),
                        key=lambda x: -float(x[1].replace(",", "") or 0))[:8]
        print("\nWarp stall reasons (warps per issued instruction):\n")
        for h, v in stalls:
            name = h.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", "")
            print(f"- {name}: {v}")
        print()
    src = ncu_csv(rep, "source", ("--print-source", "sass"))
    if len(src) > 2:
        h = src[1]
        ix = {k: i for i, k in enumerate(h)}
        cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
        by = defaultdict(lambda: defaultdict(int))
        tot = 0
        for r in src[2:]:
            if len(r) < len(h):
                continue
            op = re.sub(r"^@!?U?P\w+\s+", "", r[ix["Source"]].strip()).split(" ")[0].split(".")[0]
            for c in cols:
                try:
                    v = int(r[ix[c]] or 0)
                except ValueError:  # a second kernel's header row / non-numeric cell
                    continue
                by[op][c] += v
                tot += v
        print("Stall samples by SASS opcode (share of all samples; top reasons):\n")
        for op, dd in sorted(by.items(), key=lambda x: -sum(x[1].values()))[:10]:
            s = sum(dd.values())
            top = ", ".join(f"{k[6:]} {v / s:.0%}" for k, v in
                            sorted(dd.items(), key=lambda x: -x[1])[:3])
            print(f"- `{op}` {s / max(tot, 1):.1%} ({top})")


if __name__ == "__main__":
    main()

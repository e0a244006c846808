"""Markdown summary of one kernel in an `ncu --set full --import-source on` report.

    python tools/ncu_summary.py gpurun_out/r01_jacobi_full.ncu-rep > profiles/r01_jacobi_full.md
Key throughput / issue / memory metrics, warp-stall reasons, and the source lines
with the most stall samples (needs -lineinfo builds).
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots active %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe cycles active % (realtime)"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor memory (TMEM) cycles active %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared-memory wavefronts % of peak"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared load bank conflicts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic shared memory / CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    col = {n: i for i, n in enumerate(hdr)}
    name = vals[col["Kernel Name"]] if "Kernel Name" in col else "?"
    print(f"# ncu --set full: {name}\n\nreport: `{rep}`\n")
    print("| metric | value |\n|---|---|")
    for key, label in KEYS:
        if key in col:
            print(f"| {label} (`{key}`) | {vals[col[key]]} {units[col[key]]} |")
    stalls = []
    for n, i in col.items():
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
            try:
                stalls.append((float(vals[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1.0
    print("\n## Warp-state samples\n\n| state | share |\n|---|---|")
    for v, n in sorted(stalls, reverse=True)[:10]:
        print(f"| {n} | {100 * v / tot:.1f}% |")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
    agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
    f = line = None
    hdr2 = None
    text = ""
    for r in src:
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr2 = r
            continue
        if hdr2 is None:
            continue
        if r[0]:
            line, text = r[0], r[1]
        if len(r) > 7 and r[2]:
            try:
                smp = float(r[4].replace(",", "") or 0)
                ie = float(r[7].replace(",", "") or 0)
            except ValueError:
                continue
            a = agg[(f, line)]
            a[0] += smp
            a[1] += ie
            a[2] = text.strip()[:90]
    if agg:
        ts = sum(v[0] for v in agg.values()) or 1.0
        ti = sum(v[1] for v in agg.values()) or 1.0
        print("\n## Source lines by stall samples\n\n| samples | instructions | line | source |\n|---|---|---|---|")
        for (fn, ln), (smp, ie, t) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:20]:
            t = t.replace("|", "\\|")
            print(f"| {100 * smp / ts:.1f}% | {100 * ie / ti:.1f}% | {fn}:{ln} | `{t}` |")


if __name__ == "__main__":
    main(sys.argv[1])

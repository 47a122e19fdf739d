"""Summarise an ncu report: key throughput / occupancy metrics, stall reasons, and
instruction mix (per SASS opcode).  Usage: python tools/ncu_summary.py REPORT.ncu-rep [updates_per_launch]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
upd = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__warps_eligible.avg.per_cycle_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "sm__inst_executed.sum"]
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:60s} {vals[i]} {units[i]}")
st = [(h, vals[i]) for i, h in enumerate(hdr) if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued")]
st = sorted(st, key=lambda x: -float(x[1] or 0))[:10]
print("stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v}" for h, v in st))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
h2 = srows[1]
I, S, SRC = h2.index("Instructions Executed"), h2.index("Warp Stall Sampling (All Samples)"), h2.index("Source")
ops, stl = collections.Counter(), collections.Counter()
tot = tots = 0.0
for r in srows[2:]:
    try:
        n, s = float(r[I] or 0), float(r[S] or 0)
    except (ValueError, IndexError):
        continue
    toks = r[SRC].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    ops[op] += n
    stl[op] += s
    tot += n
    tots += s
print(f"warp instructions per launch: {tot:.4g}" + (f"  per update: {tot / upd:.1f}" if upd else ""))
print("mix:", ", ".join(f"{op} {n / tot * 100:.1f}%/{stl[op] / max(tots, 1) * 100:.1f}%" for op, n in ops.most_common(16)))

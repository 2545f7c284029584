"""Summarises an ncu --set full report of the decode kernel for profiles/ (run here, no GPU):
key raw metrics, the warp-stall breakdown and the top source lines by stall samples.
  python tools/ncu_summary.py gpurun_out/prof_TAG.ncu-rep > profiles/rNN_ncu_summary.txt"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2] if len(rows) > 2 else rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__block_size", "launch__grid_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
print(f"report: {rep}")
for w in want:
    if w in hdr:
        u = rows[1][hdr.index(w)] if len(rows) > 2 else ""
        print(f"{w:60s} {vals[hdr.index(w)]} {u}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
reasons = ['stall_long_sb', 'stall_short_sb', 'stall_wait', 'stall_mio', 'stall_selected', 'stall_branch_resolving',
           'stall_dispatch', 'stall_math', 'stall_lg', 'stall_no_inst', 'stall_barrier', 'stall_misc', 'stall_drain',
           'stall_not_selected']
tot = collections.Counter()
lines = []
h = None
cur = None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "File Path":
        cur = r[1].split('/')[-1]
        continue
    if r and r[0] == "Line No":
        h = r
        continue
    if h is None or len(r) < 40 or r[0] == "":
        continue
    d = {k: int(r[h.index(k)] or 0) for k in reasons if k in h}
    lines.append((sum(d.values()), cur, r[0], r[1].strip()[:90], max(d, key=d.get) if d else ""))
    for k, v in d.items():
        tot[k] += v
T = sum(tot.values()) or 1
print("\nwarp-stall samples by reason (share of all samples):")
for k, v in tot.most_common():
    if v:
        print(f"  {k:26s} {100 * v / T:5.1f}%")
print("\ntop source lines by stall samples:")
for x in sorted(lines, reverse=True)[:25]:
    print(f"  {100 * x[0] / T:5.1f}%  {x[1]}:{x[2]}  [{x[4]}]  {x[3]}")

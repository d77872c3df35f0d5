"""Summarise an ncu --set full report of the stepping kernel into a text file.

usage: python profiles/ncu_summary.py <report.ncu-rep> <out.txt> "<command line>" "<note>"
"""
import collections
import csv
import subprocess
import sys

rep, out, cmd, note = sys.argv[1:5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units, v = r[0], r[1], r[2]
keys = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
sr = list(csv.reader(src.splitlines()))
sh = sr[1]
ix = {k: i for i, k in enumerate(sh)}
ops = collections.Counter()
reasons = collections.Counter()
for row in sr[2:]:
    if len(row) < len(sh):
        continue
    s = row[ix["Source"]].strip()
    op = (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0] if s else "?"
    ops[op] += int(row[ix["Instructions Executed"]] or 0)
    for k in sh:
        if k.startswith("stall_") and "Not Issued" not in k:
            reasons[k] += int(row[ix[k]] or 0)
with open(out, "w") as f:
    f.write(f"command: {cmd}\nnote: {note}\n\n")
    for k in keys:
        if k in h:
            f.write(f"{k:62s} {v[h.index(k)]} {units[h.index(k)]}\n")
    tot = sum(ops.values())
    f.write("\nSASS instruction mix (executed warp-instructions):\n")
    for op, n in ops.most_common(12):
        f.write(f"  {op:10s} {100 * n / tot:5.1f}%\n")
    rs = sum(reasons.values())
    f.write("\nwarp stall samples:\n")
    for k, n in reasons.most_common(8):
        f.write(f"  {k:28s} {100 * n / rs:5.1f}%\n")
print(open(out).read())

"""Summarise an ncu report: key metrics + SASS opcode mix with stall samples."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
keys = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Avg. Not Predicated Off Threads Per Warp",
        "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput",
        "Compute (SM) Throughput", "Memory Throughput", "Grid Size", "Block Size", "Waves Per SM"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
iN, iV, iU = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
seen = set()
for r in rows[1:]:
    if r[iN] in keys and r[iN] not in seen:
        seen.add(r[iN])
        print(f"{r[iN]:45s} {r[iV]:>20s} {r[iU]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
for name in ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.sum",
             "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
             "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]:
    if name in rr[0]:
        i = rr[0].index(name)
        print(f"{name:45s} {rr[2][i]:>20s} {rr[1][i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
ops, st = collections.Counter(), collections.Counter()
tot = 0
for r in rows[2:]:
    if not r[iE].isdigit():
        continue
    toks = r[iS].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    base = op.split(".")[0]
    ops[base] += int(r[iE])
    st[base] += int(r[iW] or 0)
    tot += int(r[iE])
tst = sum(st.values()) or 1
print(f"total warp instructions {tot}")
for k, v in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"  {k:10s} {100 * v / tot:6.2f}% inst   {100 * st[k] / tst:6.2f}% stall samples")

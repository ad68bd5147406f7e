"""One invocation of the U2 (MILP DP, K4) or U3 (partition local search, K5) bench workload,
for ncu captures:  ncu -k regex:k4_dp_multi python tools/unit_kernels.py milp"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "milp"
out = bench.milp_rate(0) if what == "milp" else bench.partition_rate(0)
print(out["b200"])

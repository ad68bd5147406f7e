"""K1 device time on the bench workload for the library at GPLAN_LIB (A/B of kernel variants;
uses only the long-standing prepare/launch/collect/timing entry points)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from common import problem  # noqa: E402
from paper_2511_00796_b200.engine import Engine  # noqa: E402

p = problem("c5_1024gpu")
ids = list(range(p.cluster.n - 1))
eng = Engine(p)
eng.set_timing(True)
eng.train_prepare(ids)
k1 = []
for i in range(8):
    eng.train_launch(3, 0, -1)
    res, _ = eng.train_collect()
    k2_ms, k1_ms = eng.train_timing()
    if i >= 3:
        k1.append(k1_ms)
tag = os.environ.get("TAG", os.path.basename(os.environ.get("GPLAN_LIB", "libgplan.so")))
print(f"{tag:28s} k1 {statistics.median(k1):7.3f} ms  {res.layouts / statistics.median(k1) / 1e6:7.2f} Gcand/s  "
      f"cost {res.cost!r} rank {res.rank} feasible {res.feasible}")

"""K1 rate across train-set shapes of the C5 cluster (what the schedule's batches scan): for
type-aligned prefix sets and random subsets, device time of the K2 tables and the K1 scan per
set (median of 3 after a warm-up), candidates/s, and the type-run count R.
usage: python tools/k1_sizes.py"""
import os
import random
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from common import problem, type_prefix_sets  # noqa: E402
from paper_2511_00796_b200.engine import Engine  # noqa: E402

p = problem("c5_1024gpu")
n = p.cluster.n
sets = []
for lead in range(3):
    for m in (200, 400, 600, 800, 1000):
        sets.append((f"prefix lead={lead} m={m}", type_prefix_sets(p, lead, [m])[0]))
rng = random.Random(5)
for m in (128, 256, 512, 768, 1000):
    sets.append((f"random m={m}", sorted(rng.sample(range(n), m))))
sets.append(("bench set", list(range(n - 1))))
eng = Engine(p)
eng.set_timing(True)
print(f"{'set':28s} {'types':>5s} {'layouts':>14s} {'k2 ms':>8s} {'k1 ms':>8s} {'Gcand/s':>9s}")
for name, ids in sets:
    eng.train_prepare(ids)
    k1s, k2s = [], []
    res = None
    for i in range(4):
        eng.train_launch(3, 0, -1)
        res, _ = eng.train_collect()
        k2, k1 = eng.train_timing()
        if i:
            k1s.append(k1)
            k2s.append(k2)
    k1m, k2m = statistics.median(k1s), statistics.median(k2s)
    types = len({p.cluster.device_type[d] for d in ids})
    rate = res.layouts / ((k1m + k2m) * 1e-3) / 1e9 if res.layouts else 0
    print(f"{name:28s} {types:5d} {res.layouts:14d} {k2m:8.3f} {k1m:8.3f} {rate:9.1f}")

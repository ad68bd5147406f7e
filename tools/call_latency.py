"""Per-call latency of each C-ABI entry point (host wall clock, many calls)."""
import sys
import time

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from common import problem  # noqa: E402
from paper_2511_00796_b200 import abi  # noqa: E402
from paper_2511_00796_b200.engine import Engine  # noqa: E402

for name in sys.argv[1:] or ["c1_desk_mixed", "c3_64gpu"]:
    p = problem(name)
    eng = Engine(p)
    n = p.cluster.n
    train = list(range(0, n // 4))
    roll = list(range(n // 4, n))

    def bench(label, fn, reps=200):
        fn()
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        print(f"{name:14s} {label:22s} {1e6 * (time.perf_counter() - t) / reps:9.1f} us/call")

    bench("train_space", lambda: eng.train_space(train))
    bench("constrained_search", lambda: eng.constrained_search_raw(train, 4))
    cfgs = eng.enumerate_configs(roll)
    bench("enumerate_configs", lambda: eng.enumerate_configs(roll))
    caps = eng.rollout_capacities(roll)
    bench("solve_milp", lambda: eng.solve_milp(cfgs, caps, 256.0, p.workload.mean_len))
    res, ent = eng.solve_milp(cfgs, caps, 256.0, p.workload.mean_len)
    et = [next(t for t in range(8) if cfgs[e.config].type_counts[t] > 0) for e in ent]
    er = [e.replicas for e in ent]
    bench("weight_sync_cost", lambda: eng.weight_sync_cost(train, roll, et, er, 4))
    bench("partition_candidates", lambda: eng.partition_candidates(0.4, 0.6), reps=50)
    bench("compute_fraction", lambda: eng.partition_objective(train), reps=50)

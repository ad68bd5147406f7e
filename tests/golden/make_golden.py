"""Generates the committed golden vectors from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libref.so, i.e. `make -C oracle ref`
with /root/reference present):  python tests/golden/make_golden.py
Every fixture records the reference's own output on inputs under data/, so the
GPU box (no /root/reference) can check the oracle and the engine against it.
"""
import json
import os
import shutil
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from common import CONFIGS, ETA, problem, random_train_sets, type_prefix_sets  # noqa: E402
from oracles import Oracle, Ref, RefError  # noqa: E402

REF_PLAN = "/root/reference/proj/out/desk/plan.json"


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"))
        f.write("\n")


def main():
    shutil.copyfile(REF_PLAN, os.path.join(HERE, "desk_plan.json"))
    shutil.copyfile(REF_PLAN.replace("plan.json", "explain.txt"), os.path.join(HERE, "desk_explain.txt"))
    # ---- full schedules (plan_to_json + trace)
    sched = {}
    for name, etas in (("c1_desk_mixed", [1, -1]), ("c2_16gpu", [-1]), ("c3_64gpu", [1, 2, 3, 4])):
        ref = Ref(problem(name))
        for eta in etas:
            t = time.time()
            out = ref.schedule(eta=eta)
            sched[f"{name}/eta={eta}"] = {"plan": json.loads(out["plan_json"]), "trace": out["trace"],
                                          "ref_seconds": time.time() - t}
    dump("schedules.json", sched)
    # ---- constrained_search on sampled + probe train sets
    ts = {}
    for name in CONFIGS:
        p = problem(name)
        ref, orc = Ref(p), Oracle(p)
        n = p.cluster.n
        sets = random_train_sets(n, 24, seed=77 + n)
        for lead in range(len(p.cluster.type_names)):
            sets += type_prefix_sets(p, lead, sorted({1, 2, 3, n // 4, n // 2, n - 1}))
        cases = []
        for ids in sets:
            if orc.train_space(ids) > 300_000:  # keep the reference run bounded
                continue
            for window in (ETA[name] + 1, 2 * ETA[name] + 2):
                r = ref.constrained_search(ids, window)
                r.pop("seconds")
                cases.append({"ids": ids, "window": window, "ref": r, "layouts": orc.train_space(ids)})
        ts[name] = cases
        print(name, len(cases), "train-search cases")
    dump("train_search.json", ts)
    # ---- full candidate lists (enumeration order pin) on small sets
    cand = {}
    p = problem("c2_16gpu")
    ref = Ref(p)
    for ids in ([0, 1, 2, 3], [0, 1, 2, 8, 9], [4, 5, 6, 7, 12, 13, 14, 15], list(range(16))[::3]):
        lst = ref.train_candidates(ids, 3)
        blocks = []
        for c in lst:
            key = [s["devices"] for s in c["stages"]]
            if not blocks or blocks[-1] != key:
                blocks.append(key)
        cand[json.dumps(ids)] = {"block_lists": blocks, "candidates": lst}
    dump("train_candidates.json", cand)
    # ---- rollout side: enumerate_configs + solve_milp + weight_sync_cost on sampled rollout sets
    ro = {}
    for name in CONFIGS:
        p = problem(name)
        ref = Ref(p)
        n = p.cluster.n
        cases = []
        for train in random_train_sets(n, 30, seed=500 + n):
            roll = sorted(set(range(n)) - set(train))
            window = ETA[name] + 1
            cfg = ref.enumerate_configs(roll)
            states = 1
            for c in cfg["capacities"]:
                states *= c + 1
            if states > 400_000:
                continue
            case = {"train": train, "rollout": roll, "window": window, "configs": cfg["configs"],
                    "capacities": cfg["capacities"]}
            B = float(p.workload.batch_rollouts * window)
            try:
                plan = ref.solve_milp(cfg["configs"], cfg["capacities"], B, p.workload.mean_len)
                plan.pop("seconds")
                case["milp"] = plan
                case["weight_sync"] = ref.weight_sync(train, roll, window, plan)
            except RefError as e:
                case["milp_error"] = e.code
            cases.append(case)
        ro[name] = cases
        print(name, len(cases), "rollout cases")
    dump("rollout.json", ro)
    # ---- graph_partition_candidates: scheduler-style probes (top-8, gamma grid, widened bands)
    parts = {}
    for name in CONFIGS + ["t10_tiny", "t8_tiny"]:
        p = problem(name)
        ref = Ref(p)
        cases = []
        grid = [1, 4, 8, 12, 15] if name == "c5_1024gpu" else range(1, 16)
        for pp in grid:
            gm = pp / 16
            for widen in (0.0, 0.05):
                for machine in ((False, True) if name != "c5_1024gpu" else (False,)):
                    lo, hi = max(0.0, gm - widen), min(1.0, gm + widen)
                    case = {"gamma_l": lo, "gamma_h": hi, "machine": machine}
                    try:
                        out = ref.partition_candidates(lo, hi, k=8, seed=4276115, machine=machine)
                        case["candidates"] = out["candidates"]
                    except RefError as e:
                        case["error"] = e.code
                    cases.append(case)
        if name in ("t10_tiny", "t8_tiny"):  # heuristic tier on exact-size clusters
            for lo, hi in ((0.2, 0.5), (0.4, 0.7), (0.1, 0.9)):
                out = ref.partition_candidates(lo, hi, k=8, seed=99, force_local=True)
                cases.append({"gamma_l": lo, "gamma_h": hi, "machine": False, "force_local": True,
                              "seed": 99, "candidates": out["candidates"]})
        parts[name] = cases
        print(name, len(cases), "partition cases")
    dump("partition.json", parts)


if __name__ == "__main__":
    main()

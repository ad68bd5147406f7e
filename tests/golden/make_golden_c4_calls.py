"""Reference goldens for a seeded sample of the seam calls the C4 schedule() makes.

The reference's own C4 schedule() takes hours, so the call list was recorded
from the UNMODIFIED reference scheduler running on the engine through the drop-in shim —
on a GPU box:

    GPLAN_SHIM_LOG=gpurun_out/c4_calls.jsonl \
    LD_PRELOAD=paper_2511_00796_b200/libgplan_shim.so python tests/dropin_driver.py c4_256gpu/eta=2

— and every sampled call is then answered here by the UNMODIFIED reference
(oracle/_ref/libref.so) on the host cores:

    python tests/golden/make_golden_c4_calls.py gpurun_out/c4_calls.jsonl

Sample (seed 2511): every distinct graph_partition_candidates band; 60 evaluate_partition
triples (constrained_search + enumerate_configs + solve_milp, + weight_sync_cost) drawn
10 per decade of the train set's layout count (1e0 .. 1e6, the largest ~3.4e6); 20 more
solve_milp calls drawn from the largest capacity lattices. tests/test_engine_c4_calls.py
checks the engine against all of them.
"""
import json
import math
import multiprocessing as mp
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from common import problem  # noqa: E402
from oracles import Oracle, Ref, RefError  # noqa: E402

NAME = "c4_256gpu"


def triples(log):
    out = []
    for i, x in enumerate(log):
        if x["call"] == "constrained_search":
            e, m = log[i + 1], log[i + 2]
            assert e["call"] == "enumerate_configs" and m["call"] == "solve_milp"
            out.append({"train": x["ids"], "window": x["window"], "rollout": e["ids"],
                        "total_rollouts": m["total_rollouts"], "mean_len": m["mean_len"], "caps": m["caps"]})
    return out


def answer_eval(t):
    p = problem(NAME)
    ref = Ref(p)
    t0 = time.time()
    out = dict(t)
    out["train_ref"] = ref.constrained_search(t["train"], t["window"])
    out["train_ref"].pop("seconds", None)
    cfg = ref.enumerate_configs(t["rollout"])
    out["configs"] = cfg["configs"]
    assert cfg["capacities"] == t["caps"]
    try:
        plan = ref.solve_milp(cfg["configs"], t["caps"], t["total_rollouts"], t["mean_len"])
        plan.pop("seconds", None)
        out["milp"] = plan
        if out["train_ref"]["found"]:
            out["weight_sync"] = ref.weight_sync(t["train"], t["rollout"], t["window"], plan)
    except RefError as e:
        out["milp_error"] = e.code
    out["ref_seconds"] = time.time() - t0
    return out


def answer_part(b):
    ref = Ref(problem(NAME))
    out = dict(b)
    try:
        r = ref.partition_candidates(b["gamma_l"], b["gamma_h"], k=b["k"], seed=b["seed"], restarts=b["restarts"],
                                     q=b["q"], r=b["r"], force_local=bool(b["force_local"]),
                                     machine=bool(b["machine"]))
        out["candidates"] = r["candidates"]
    except RefError as e:
        out["error"] = e.code
    return out


def main(path):
    log = [json.loads(x) for x in open(path)]
    orc = Oracle(problem(NAME))
    rng = random.Random(2511)
    tri = triples(log)
    by_dec = {}
    for t in tri:
        by_dec.setdefault(int(math.log10(max(1, orc.train_space(t["train"])))), []).append(t)
    sample = []
    for d in sorted(by_dec):
        sample += rng.sample(by_dec[d], min(10, len(by_dec[d])))
    rest = [t for t in tri if t not in sample]
    rest.sort(key=lambda t: -math.prod(c + 1 for c in t["caps"]))
    sample += rest[:20]
    bands, seen = [], set()
    for x in log:
        if x["call"] == "graph_partition_candidates":
            key = (x["q"], x["r"], x["gamma_l"], x["gamma_h"])
            if key not in seen:
                seen.add(key)
                bands.append({k: x[k] for k in ("q", "r", "gamma_l", "gamma_h", "k", "seed", "restarts",
                                                "exact_threshold", "force_local", "machine")})
    with mp.Pool(min(6, os.cpu_count() or 1)) as pool:
        evals = pool.map(answer_eval, sorted(sample, key=lambda t: -orc.train_space(t["train"])), chunksize=1)
        parts = pool.map(answer_part, bands, chunksize=1)
    with open(os.path.join(HERE, "c4_calls.json"), "w") as f:
        json.dump({"config": NAME, "eta": 2, "calls_logged": len(log), "evaluations": evals, "partitions": parts},
                  f, separators=(",", ":"))
        f.write("\n")
    print(len(evals), "evaluations,", len(parts), "partition calls")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c4_calls.jsonl")

"""GPU parity: the sm_100a layout search vs the oracle / the reference's golden vectors.

Bar (BASELINE.json north_star): selected plan, feasible-set size and cost
bit-exact (cost compared with ==, not a tolerance).
"""
import pytest

from common import CONFIGS, ETA, golden, problem, random_train_sets, type_prefix_sets
from oracles import Oracle, train_result_dict

pytestmark = pytest.mark.gpu

_engines = {}


def engine(name):
    from paper_2511_00796_b200.engine import Engine
    if name not in _engines:
        _engines[name] = Engine(problem(name))
    return _engines[name]


def run(name, ids, window, lo=0, hi=-1):
    res, devs = engine(name).constrained_search_raw(ids, window, lo=lo, hi=hi)
    return train_result_dict(res, devs)


@pytest.mark.parametrize("name", CONFIGS)
def test_golden_train_search(name):
    for case in golden("train_search.json")[name]:
        got = run(name, case["ids"], case["window"])
        ref = case["ref"]
        assert got["found"] == ref["found"], case["ids"]
        assert got["layouts"] == case["layouts"]
        if ref["found"]:
            assert got["cost"] == ref["cost"], case["ids"]
            assert got["stages"] == ref["stages"], case["ids"]


@pytest.mark.parametrize("name", CONFIGS[:4])
def test_random_sets_vs_oracle(name):
    p = problem(name)
    orc = Oracle(p)
    sets = random_train_sets(p.cluster.n, 40, seed=1000 + p.cluster.n)
    for lead in range(len(p.cluster.type_names)):
        sets += type_prefix_sets(p, lead, range(1, p.cluster.n, max(1, p.cluster.n // 12)))
    checked = 0
    for ids in sets:
        if orc.train_space(ids) > 200_000:
            continue
        for window in (1, ETA[name] + 1, 64):
            want = orc.constrained_search(ids, window)
            got = run(name, ids, window)
            assert got == want, (ids, window)
            checked += 1
    assert checked >= 40


def test_ranges_recombine_exactly():
    """Rank-range sharding (multi-GPU split): lexicographic (cost, rank) min over shards == full."""
    name = "c4_256gpu"
    p = problem(name)
    eng = engine(name)
    ids = list(range(1, p.cluster.n))
    total = eng.train_space(ids)
    assert total > 1_000_000
    full = run(name, ids, 3)
    shards = [(total * i) // 8 for i in range(9)]
    parts = [run(name, ids, 3, lo=a, hi=b) for a, b in zip(shards, shards[1:])]
    assert sum(x["feasible"] for x in parts) == full["feasible"]
    assert sum(x["layouts"] for x in parts) == total
    win = min((x for x in parts if x["found"]), key=lambda x: (x["cost"], x["rank"]))
    assert win == {**full, "layouts": win["layouts"], "feasible": win["feasible"]}
    # a window of the space deep inside, checked against the oracle restricted to it
    lo, hi = total // 3, total // 3 + 50_000
    assert run(name, ids, 3, lo=lo, hi=hi) == Oracle(p).constrained_search(ids, 3, lo=lo, hi=hi)


def test_c5_full_space_slices_vs_oracle():
    """C5 (1024 GPUs, 3 types): a 2.4e9-layout train set; slices checked against the oracle."""
    name = "c5_1024gpu"
    p = problem(name)
    ids = list(range(p.cluster.n))[:-1]
    eng = engine(name)
    total = eng.train_space(ids)
    assert total == Oracle(p).train_space(ids)
    assert total > 2_000_000_000
    orc = Oracle(p)
    for lo in (0, total // 7, total // 2, total - 40_000):
        hi = min(total, lo + 40_000)
        assert run(name, ids, 3, lo=lo, hi=hi) == orc.constrained_search(ids, 3, lo=lo, hi=hi)


def test_edge_cases():
    from paper_2511_00796_b200 import abi
    from paper_2511_00796_b200.engine import ValidationError
    eng = engine("c5_1024gpu")
    with pytest.raises(ValidationError):
        eng.constrained_search([], 3)
    with pytest.raises(ValidationError):
        eng.constrained_search([0, 0], 3)
    with pytest.raises(ValidationError):
        eng.constrained_search([5000], 3)
    with pytest.raises(ValidationError):
        eng.constrained_search([0, 1], 3, opts=abi.gp_train_opts(5, 16))
    # 70B on one H800: nothing fits -> std::nullopt, same as the oracle
    assert eng.constrained_search([0], 3) is None
    orc = Oracle(problem("c5_1024gpu"))
    assert orc.constrained_search([0], 3)["found"] is False
    # single device that fits
    got = run("c1_desk_mixed", [3], 2)
    assert got == Oracle(problem("c1_desk_mixed")).constrained_search([3], 2)


def test_multi_gpu_context_fanout():
    """gp_ctx_create_multi: one search split over every visible GPU == the single-GPU result.
    On a one-GPU box the context holds two peer contexts on device 0 (same fan-out, shard
    reduction and host merge code, sharing one GPU)."""
    import torch
    n = torch.cuda.device_count()
    from paper_2511_00796_b200.engine import Engine
    p = problem("c5_1024gpu")
    multi = Engine(p, devices=list(range(n)) if n >= 2 else [0, 0])
    ids = list(range(p.cluster.n))[:-1]
    # a 1.8e8-layout sub-range, large enough to fan out
    lo, hi = 100_000_000, 280_000_000
    r1, d1 = engine("c5_1024gpu").constrained_search_raw(ids, 3, lo=lo, hi=hi)
    r2, d2 = multi.constrained_search_raw(ids, 3, lo=lo, hi=hi)
    assert train_result_dict(r1, d1) == train_result_dict(r2, d2)


def test_memo_window_sweep_vs_oracle():
    """One scan per train set answers every window: repeated searches of the same sets
    with windows 1..70 (memo hits after the first) == the oracle, and == a memo-less context."""
    from paper_2511_00796_b200.engine import Engine
    name = "c3_64gpu"
    p = problem(name)
    orc = Oracle(p)
    memo_less = Engine(p)
    memo_less.set_memo(False)
    sets = [s for s in random_train_sets(p.cluster.n, 30, seed=77) if orc.train_space(s) <= 60_000][:8]
    assert len(sets) >= 4
    for ids in sets:
        for window in (3, 1, 2, 6, 7, 12, 24, 33, 48, 64, 70):
            want = orc.constrained_search(ids, window)
            assert run(name, ids, window) == want, (ids, window)
            r, d = memo_less.constrained_search_raw(ids, window)
            assert train_result_dict(r, d) == want, (ids, window)


def test_generic_scan_fractional_flops():
    """Fractional FLOPS (the reference's random_instance style, tests/test_fixtures.cpp:108):
    allocate_layers' total then depends on the layout's grouping, K1-fast does not apply,
    and the generic scan must still equal the oracle."""
    import json

    from common import read
    from paper_2511_00796_b200 import load_problem
    from paper_2511_00796_b200.engine import Engine
    doc = json.loads(read("clusters", "c3_64gpu"))
    for i, t in enumerate(doc["gpu_types"]):
        t["flops_tflops"] = t["flops_tflops"] * (1.0 + 0.0123456789 * (i + 1)) + 0.1
    p = load_problem(json.dumps(doc), read("workloads", "c3_64gpu"), read("calibration", "c3_64gpu"))
    orc = Oracle(p)
    eng = Engine(p)
    sets = [s for s in random_train_sets(p.cluster.n, 40, seed=4242) if orc.train_space(s) <= 100_000][:12]
    assert len(sets) >= 6
    for ids in sets:
        for window in (1, 2, 33):
            res, devs = eng.constrained_search_raw(ids, window)
            assert train_result_dict(res, devs) == orc.constrained_search(ids, window), (ids, window)


def test_fast_scan_equals_generic_scan(monkeypatch):
    """K1-fast vs the generic K1 (GPLAN_K1_GENERIC=1) on large ranges: same winner, cost and
    feasible count (every candidate is scored, by the tables or by the generic fallback)."""
    for name, span in (("c4_256gpu", None), ("c5_1024gpu", 30_000_000)):
        p = problem(name)
        eng = engine(name)
        ids = list(range(1, p.cluster.n))
        total = eng.train_space(ids)
        lo, hi = (0, total) if span is None else (total // 3, total // 3 + span)
        fast = run(name, ids, 3, lo=lo, hi=hi)
        monkeypatch.setenv("GPLAN_K1_GENERIC", "1")
        generic = run(name, ids, 3, lo=lo, hi=hi)
        monkeypatch.delenv("GPLAN_K1_GENERIC")
        assert fast == generic, name


def test_device_level_links_path(monkeypatch):
    """K2a/K2b over device pairs (GPLAN_DEVICE_LINKS=1) == over machine pairs (default,
    certified at context creation) == the oracle."""
    from paper_2511_00796_b200.engine import Engine
    name = "c3_64gpu"
    p = problem(name)
    orc = Oracle(p)
    monkeypatch.setenv("GPLAN_DEVICE_LINKS", "1")
    dev_level = Engine(p)
    monkeypatch.delenv("GPLAN_DEVICE_LINKS")
    sets = [s for s in random_train_sets(p.cluster.n, 30, seed=2024) if orc.train_space(s) <= 100_000][:8]
    for ids in sets:
        want = orc.constrained_search(ids, 3)
        r, d = dev_level.constrained_search_raw(ids, 3)
        assert train_result_dict(r, d) == want, ids
        assert run(name, ids, 3) == want, ids


def test_four_type_runs(monkeypatch):
    """Four GPU types (the R = 4 instantiations of K1 and K1-fast): a 6.9e7-layout set —
    fast == generic on the full range, slices == the oracle — and random subsets == oracle."""
    name = "t4types_288gpu"
    p = problem(name)
    orc = Oracle(p)
    ids = list(range(p.cluster.n))
    total = engine(name).train_space(ids)
    assert total == orc.train_space(ids) and total > 1 << 20
    _, fast_used = engine(name).debug_layout_costs(ids, 0, 4096, path=0)
    assert fast_used == 4  # K1-fast, the last of the 4 type runs innermost
    fast = run(name, ids, 3, lo=0, hi=total)
    monkeypatch.setenv("GPLAN_K1_GENERIC", "1")
    generic = run(name, ids, 3, lo=0, hi=total)
    monkeypatch.delenv("GPLAN_K1_GENERIC")
    assert fast == generic
    for lo in (0, total // 5, total // 2, total - 30_000):
        hi = min(total, lo + 30_000)
        assert run(name, ids, 3, lo=lo, hi=hi) == orc.constrained_search(ids, 3, lo=lo, hi=hi)
    checked = 0
    for s in random_train_sets(p.cluster.n, 40, seed=4444, max_size=48):
        if orc.train_space(s) > 150_000:
            continue
        assert run(name, s, 2) == orc.constrained_search(s, 2), s
        checked += 1
    assert checked >= 5


def test_deferred_and_overflow_paths(monkeypatch):
    """K1-fast's generic fallback: with every candidate deferred (test hook), a range that
    fits the device queue is scored by k1_deferred, a larger one overflows it and is rescanned
    by the generic K1 — both equal to the normal scan."""
    name = "c5_1024gpu"
    p = problem(name)
    ids = list(range(p.cluster.n))[:-1]
    total = engine(name).train_space(ids)
    for lo, hi in ((total // 4, total // 4 + 1_500_000), (total // 2, total // 2 + 3_000_000)):
        want = run(name, ids, 3, lo=lo, hi=hi)
        assert want["feasible"] > 0
        monkeypatch.setenv("GPLAN_K1_DEFER_ALL", "1")
        got = run(name, ids, 3, lo=lo, hi=hi)
        monkeypatch.delenv("GPLAN_K1_DEFER_ALL")
        assert got == want, (lo, hi)

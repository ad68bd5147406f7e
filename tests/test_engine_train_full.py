"""GPU: constrained_search at full C4/C5 scale against the independent CPU restatement.

* Whole-space winners: every set of tests/golden/train_full.json (incl. the 2.42e9-layout
  C5 bench set) — (cost, rank) for windows 1..8 and the memory-feasible count equal the
  table-memoised C restatement's (oracle.c or_constrained_search_tab, pinned against the
  reference goldens by tests/golden/make_golden_full.py and test_oracle.py).
* K1-fast == generic K1 over the FULL bench set (every window, feasible count).
* Per-candidate per_step (north_star: "per-candidate cost estimates match"): the scan
  kernel's own value (DUMP instantiation, K1-fast path active) equals the oracle's
  bit-for-bit on >= 1e5 random ranks per set, on the ranks around the bench winner and
  around every golden window winner; the deferred (generic) fallback and the generic K1
  agree on the same ranks.
Reference: src/train_search.cpp:218-275, src/cost_model.cpp:93-126.
"""
import os

import numpy as np
import pytest

from common import golden, problem
from oracles import Oracle

pytestmark = pytest.mark.gpu

FULL = golden("train_full.json")
WINDOWS = list(range(1, 9))


def _cases(name):
    return [(name, i) for i in range(len(FULL[name]))]


@pytest.fixture(scope="module")
def engines():
    from paper_2511_00796_b200.engine import Engine
    out = {n: Engine(problem(n)) for n in ("c4_256gpu", "c5_1024gpu")}
    yield out
    for e in out.values():
        e.close()


@pytest.mark.parametrize("name,i", _cases("c4_256gpu") + _cases("c5_1024gpu"))
def test_full_space_winner_matches_oracle(engines, name, i):
    case = FULL[name][i]
    eng = engines[name]
    for w in WINDOWS:
        res, _ = eng.constrained_search_raw(case["ids"], w)
        want = case["windows"][str(w)]
        assert res.layouts == case["layouts"]
        assert res.feasible == case["feasible"]
        if want["rank"] < 0:
            assert not res.found
        else:
            assert (res.cost, res.rank) == (want["cost"], want["rank"]), (w, res.cost, res.rank, want)


def test_fast_equals_generic_on_full_bench_set(engines):
    eng = engines["c5_1024gpu"]
    ids = FULL["c5_1024gpu"][0]["ids"]
    assert len(ids) == 1023
    eng.set_memo(False)
    try:
        fast = [eng.constrained_search_raw(ids, w, lo=0, hi=-1)[0] for w in (1, 3, 7)]
        os.environ["GPLAN_K1_GENERIC"] = "1"
        try:
            gen = [eng.constrained_search_raw(ids, w, lo=0, hi=-1)[0] for w in (1, 3, 7)]
        finally:
            del os.environ["GPLAN_K1_GENERIC"]
    finally:
        eng.set_memo(True)
    for a, b in zip(fast, gen):
        assert (a.found, a.cost, a.rank, a.feasible, a.layouts) == (b.found, b.cost, b.rank, b.feasible, b.layouts)
        assert a.layouts == 2_415_919_104


def _ranges(total, rng, n_windows, width, anchors):
    out = []
    for a in anchors:
        lo = max(0, min(total - width, a - width // 2))
        out.append((lo, lo + width))
    for lo in rng.integers(0, total - width, size=n_windows):
        out.append((int(lo), int(lo) + width))
    return sorted(set(out))


@pytest.mark.parametrize("name,i", [("c5_1024gpu", 0), ("c5_1024gpu", 8), ("c4_256gpu", 0), ("c4_256gpu", 7)])
def test_per_candidate_costs_vs_oracle(engines, name, i):
    """path 0: the whole-space scan a search runs (K1-fast), values of the ranks kept; path 3:
    K1-fast on the ranges themselves; path 1: generic K1; path 2: every candidate through
    K1-fast's deferred fallback."""
    case = FULL[name][i]
    eng, orc = engines[name], Oracle(problem(name))
    ids, total = case["ids"], case["layouts"]
    rng = np.random.default_rng(1234 + i)
    anchors = sorted({v["rank"] for v in case["windows"].values() if v["rank"] >= 0})
    rs = _ranges(total, rng, 50, 2048, anchors)
    want = orc.layout_costs_tab(ids, rs)
    got, inner = [], set()
    for lo, hi in rs:
        v, fast = eng.debug_layout_costs(ids, lo, hi, path=0)
        got.append(v)
        inner.add(fast)
    got = np.concatenate(got)
    assert inner == {3}  # K1-fast (constant allocation total), the last of the 3 type runs innermost
    assert got.size >= 100_000
    assert not np.isnan(got).any()
    np.testing.assert_array_equal(got.view(np.int64), want.view(np.int64))  # bitwise
    assert np.isfinite(got).sum() > 0
    # the plain (un-memoised) restatement on a subset
    for lo, hi in rs[:4]:
        plain = orc.layout_costs(ids, lo, hi)
        tab = orc.layout_costs_tab(ids, [(lo, hi)])
        np.testing.assert_array_equal(plain.view(np.int64), tab.view(np.int64))
    # range scans, generic K1 and K1-fast's deferred (generic) fallback on the same ranks
    sub = rs[:12]
    want_sub = orc.layout_costs_tab(ids, sub)
    for path in (3, 1, 2):
        g = np.concatenate([eng.debug_layout_costs(ids, lo, hi, path=path)[0] for lo, hi in sub])
        np.testing.assert_array_equal(g.view(np.int64), want_sub.view(np.int64))


@pytest.mark.parametrize("n_shards", [2, 3, 8])
def test_shards_recombine_to_the_whole_space(engines, n_shards):
    """gp_train_shard_bounds + one range search per shard (what bench.py's ranks and the
    multi-GPU fan-out run): winners merged by (cost, rank) and feasible counts summed ==
    the whole-space search, for every window."""
    eng = engines["c5_1024gpu"]
    case = FULL["c5_1024gpu"][0]
    b = eng.shard_bounds(case["ids"], n_shards)
    assert b[0] == 0 and b[-1] == case["layouts"] and all(x <= y for x, y in zip(b, b[1:]))
    for w in (1, 3):
        best, feas = None, 0
        for lo, hi in zip(b, b[1:]):
            r, _ = eng.constrained_search_raw(case["ids"], w, lo=lo, hi=hi)
            feas += r.feasible
            if r.found and (best is None or (r.cost, r.rank) < best):
                best = (r.cost, r.rank)
        want = case["windows"][str(w)]
        assert best == (want["cost"], want["rank"]) and feas == case["feasible"]


@pytest.mark.parametrize("lead,m", [(0, 780), (0, 800), (1, 790), (1, 830), (2, 790)])
def test_small_last_run_sets_vs_oracle(engines, lead, m):
    """Type-aligned prefix probes whose last type run is one to a few machines (a handful of
    last-run choices per prefix): the generic scan with one prefix per lane
    (k1_layout_scan_grouped<R, 1>) gives the restatement's winner for windows 1..4 and its
    feasible count; 4-lane groups (GPLAN_K1_GROUP=4) and one prefix per warp
    (GPLAN_K1_UNGROUPED=1) agree; per-candidate values through the grouped DUMP kernel equal
    the oracle's on random ranges."""
    from common import type_prefix_sets
    p = problem("c5_1024gpu")
    eng, orc = engines["c5_1024gpu"], Oracle(p)
    ids = type_prefix_sets(p, lead, [m])[0]
    wins = [1, 2, 3, 4]
    o = orc.constrained_search_tab(ids, wins)
    want, feas, lay = o["windows"], o["feasible"], o["layouts"]
    eng.set_memo(False)
    try:
        got = {w: eng.constrained_search_raw(ids, w)[0] for w in wins}
        os.environ["GPLAN_K1_UNGROUPED"] = "1"
        try:
            plain = {w: eng.constrained_search_raw(ids, w)[0] for w in wins}
        finally:
            del os.environ["GPLAN_K1_UNGROUPED"]
        os.environ["GPLAN_K1_GROUP"] = "4"
        try:
            grp4 = {w: eng.constrained_search_raw(ids, w)[0] for w in wins}
        finally:
            del os.environ["GPLAN_K1_GROUP"]
    finally:
        eng.set_memo(True)
    for w in wins:
        r = got[w]
        assert (r.layouts, r.feasible) == (lay, feas)
        assert (r.cost, r.rank) == want[w], (w, r.cost, r.rank, want[w])
        assert (plain[w].cost, plain[w].rank, plain[w].feasible) == (r.cost, r.rank, r.feasible)
        assert (grp4[w].cost, grp4[w].rank, grp4[w].feasible) == (r.cost, r.rank, r.feasible)
    rng = np.random.default_rng(m)
    rs = _ranges(lay, rng, 8, 4096, [want[w][1] for w in wins if want[w][1] >= 0])
    ref = orc.layout_costs_tab(ids, rs)
    g = np.concatenate([eng.debug_layout_costs(ids, lo, hi, path=1)[0] for lo, hi in rs])
    np.testing.assert_array_equal(g.view(np.int64), ref.view(np.int64))

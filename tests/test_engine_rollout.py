"""GPU parity of the rollout side: K3 configs, K4 MILP DP, K6 weight sync (bit-exact)."""
import random

import pytest

from common import CONFIGS, ETA, golden, problem, random_train_sets
from oracles import Oracle, config_dict, oracle_configs, oracle_milp, oracle_weight_sync

pytestmark = pytest.mark.gpu
_engines = {}


def engine(name):
    from paper_2511_00796_b200.engine import Engine
    if name not in _engines:
        _engines[name] = Engine(problem(name))
    return _engines[name]


def check_rollout(name, roll, window, train=None, max_states=2_000_000):
    p = problem(name)
    eng, orc = engine(name), Oracle(p)
    T = len(p.cluster.type_names)
    got = eng.enumerate_configs(roll)
    want = oracle_configs(orc, roll)
    assert [config_dict(c, T) for c in got] == [config_dict(c, T) for c in want]
    caps = eng.rollout_capacities(roll)
    states = 1
    for c in caps:
        states *= c + 1
    if states > max_states or not got:
        return None
    B = float(p.workload.batch_rollouts * window)
    rc, res_o, ent_o = oracle_milp(orc, want, caps, B, p.workload.mean_len)
    from paper_2511_00796_b200.engine import InfeasibleError
    if rc:
        with pytest.raises(InfeasibleError):
            eng.solve_milp(got, caps, B, p.workload.mean_len)
        return None
    res, ent = eng.solve_milp(got, caps, B, p.workload.mean_len)
    assert res.makespan == res_o.makespan and res.aggregate == res_o.aggregate
    assert [(e.config, e.replicas, e.workload) for e in ent] == \
        [(e.config, e.replicas, e.workload) for e in ent_o]
    if train is not None:
        et = [next(t for t in range(T) if got[e.config].type_counts[t] > 0) for e in ent]
        er = [e.replicas for e in ent]
        assert eng.weight_sync_cost(train, roll, et, er, window) == \
            oracle_weight_sync(orc, train, roll, et, er, window)
    return states


@pytest.mark.parametrize("name", CONFIGS)
def test_golden_rollout(name):
    p = problem(name)
    eng = engine(name)
    T = len(p.cluster.type_names)
    for case in golden("rollout.json")[name]:
        cfgs = eng.enumerate_configs(case["rollout"])
        assert [config_dict(c, T) for c in cfgs] == \
            [{k: c[k] for k in ("type_counts", "tp_per_stage", "throughput")} for c in case["configs"]]
        if "milp" not in case:
            continue
        B = float(p.workload.batch_rollouts * case["window"])
        res, ent = eng.solve_milp(cfgs, case["capacities"], B, p.workload.mean_len)
        m = case["milp"]
        assert res.makespan == m["makespan"]
        assert [(e.replicas, e.workload) for e in ent] == [(e["replicas"], e["workload"]) for e in m["entries"]]
        et = [next(t for t in range(T) if cfgs[e.config].type_counts[t] > 0) for e in ent]
        er = [e.replicas for e in ent]
        assert eng.weight_sync_cost(case["train"], case["rollout"], et, er, case["window"]) == case["weight_sync"]


@pytest.mark.parametrize("name", CONFIGS[:4])
def test_random_rollout_sets_vs_oracle(name):
    p = problem(name)
    n = p.cluster.n
    checked = 0
    for train in random_train_sets(n, 25, seed=900 + n):
        roll = sorted(set(range(n)) - set(train))
        if check_rollout(name, roll, ETA[name] + 1, train=train):
            checked += 1
    assert checked >= 5


def test_large_lattice_c5():
    """C5-scale rollout sets: multi-million-state lattices, 3 types (oracle-checked)."""
    p = problem("c5_1024gpu")
    rng = random.Random(7)
    cl = p.cluster
    done = 0
    for _ in range(6):
        roll = sorted(rng.sample(range(cl.n), rng.randint(60, 180)))
        if check_rollout("c5_1024gpu", roll, 3, max_states=3_000_000):
            done += 1
    assert done >= 3


def test_milp_errors():
    from paper_2511_00796_b200.engine import InfeasibleError, ValidationError
    eng = engine("c3_64gpu")
    p = problem("c3_64gpu")
    cfgs = eng.enumerate_configs(list(range(64)))
    with pytest.raises(ValidationError):  # lattice > 5e7 (src/rollout_milp.cpp:110-112)
        eng.solve_milp(cfgs, [400, 400, 400], 64.0, p.workload.mean_len)
    with pytest.raises(InfeasibleError):  # no configs
        eng.solve_milp([], [8, 8, 8], 64.0, p.workload.mean_len)
    res, ent = eng.solve_milp(cfgs, [8, 8, 8], 0.0, p.workload.mean_len)  # B <= 0: empty plan
    assert res.n_entries == 0 and ent == []
    with pytest.raises(ValidationError):
        eng.enumerate_configs([])


@pytest.mark.parametrize("name", ["c3_64gpu", "c4_256gpu", "c5_1024gpu"])
def test_milp_batch_vs_oracle(name):
    """gp_solve_milp_batch: many rollout sets (distinct config lists, nested and unrelated
    lattices) solved in one call — the lattice DPs of all new tables in one launch — each
    equal to the oracle's solve_milp."""
    from paper_2511_00796_b200.engine import Engine
    p = problem(name)
    eng, orc = Engine(p), Oracle(p)
    n = p.cluster.n
    rng = random.Random(4040 + n)
    queries, wants = [], []
    B = float(p.workload.batch_rollouts * 3)
    for train in random_train_sets(n, 40, seed=4040 + n):
        roll = sorted(set(range(n)) - set(train))
        if n > 256:
            roll = sorted(rng.sample(range(n), rng.randint(40, 140)))
        cfgs = eng.enumerate_configs(roll)
        caps = eng.rollout_capacities(roll)
        states = 1
        for c in caps:
            states *= c + 1
        if not cfgs or states > 2_000_000:
            continue
        queries.append((cfgs, list(caps)))
        wants.append(oracle_milp(orc, oracle_configs(orc, roll), caps, B, p.workload.mean_len))
    assert len(queries) >= 8
    got = eng.solve_milp_batch(queries, B)
    for (st, res, ent), (rc, res_o, ent_o) in zip(got, wants):
        assert (st == 0) == (rc == 0)
        if rc == 0:
            assert res.makespan == res_o.makespan and res.aggregate == res_o.aggregate
            assert [(e.config, e.replicas, e.workload) for e in ent] == \
                [(e.config, e.replicas, e.workload) for e in ent_o]


@pytest.mark.parametrize("name", ["c3_64gpu", "c5_1024gpu"])
def test_rollout_max_stages_up_to_8(name):
    """RolloutSearchOptions::max_stages 1..8 (GP_MAX_ROLLOUT_STAGES): K3's config lists equal
    the oracle's and the unmodified reference's (src/rollout_milp.cpp:39-89), and the MILP
    over the deeper configs equals the oracle's; > 8 is rejected (gp_config holds 8 stages)."""
    from oracles import Ref, ref_available

    from paper_2511_00796_b200 import abi
    from paper_2511_00796_b200.engine import ValidationError
    p = problem(name)
    eng, orc = engine(name), Oracle(p)
    T = len(p.cluster.type_names)
    ref = Ref(p) if ref_available() else None
    n = p.cluster.n
    sets = [sorted(set(range(n)) - set(t)) for t in random_train_sets(n, 4, seed=31 + n)]
    sets.append(list(range(n)))
    for roll in sets:
        for ms in range(1, 9):
            got = [config_dict(c, T) for c in eng.enumerate_configs(roll, opts=abi.gp_rollout_opts(ms))]
            assert got == [config_dict(c, T) for c in oracle_configs(orc, roll, max_stages=ms)], ms
            if ref is not None:
                want = ref.enumerate_configs(roll, max_stages=ms)["configs"]
                assert got == [{k: c[k] for k in ("type_counts", "tp_per_stage", "throughput")} for c in want]
        with pytest.raises(ValidationError):
            eng.enumerate_configs(roll, opts=abi.gp_rollout_opts(9))
    roll = sets[0]
    cfgs = eng.enumerate_configs(roll, opts=abi.gp_rollout_opts(8))
    caps = eng.rollout_capacities(roll)
    states = 1
    for c in caps:
        states *= c + 1
    if states <= 3_000_000:
        B = float(p.workload.batch_rollouts * 3)
        rc, res_o, ent_o = oracle_milp(orc, oracle_configs(orc, roll, max_stages=8), caps, B, p.workload.mean_len)
        assert rc == 0
        res, ent = eng.solve_milp(cfgs, caps, B, p.workload.mean_len)
        assert res.makespan == res_o.makespan
        assert [(e.config, e.replicas, e.workload) for e in ent] == \
            [(e.config, e.replicas, e.workload) for e in ent_o]

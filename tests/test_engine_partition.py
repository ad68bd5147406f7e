"""GPU parity of the repartition solver (K5): exact tier and restart local search, bit-exact."""
import pytest

from common import CONFIGS, golden, problem
from oracles import Oracle, oracle_partitions

pytestmark = pytest.mark.gpu
_engines = {}


def engine(name):
    from paper_2511_00796_b200.engine import Engine
    if name not in _engines:
        _engines[name] = Engine(problem(name))
    return _engines[name]


def run(name, lo, hi, seed=4276115, force_local=False, machine=False, restarts=16, k=8):
    from paper_2511_00796_b200 import abi
    o = abi.gp_part_opts(12, restarts, seed, 1e-9, int(force_local), int(machine))
    return engine(name).partition_candidates(lo, hi, k=k, opts=o)


@pytest.mark.parametrize("name", CONFIGS + ["t10_tiny", "t8_tiny"])
def test_golden_partitions(name):
    from paper_2511_00796_b200.engine import BandInfeasibleError
    for case in golden("partition.json")[name]:
        kw = dict(seed=case.get("seed", 4276115), force_local=case.get("force_local", False),
                  machine=case["machine"])
        if "error" in case:
            with pytest.raises(BandInfeasibleError):
                run(name, case["gamma_l"], case["gamma_h"], **kw)
            continue
        got = run(name, case["gamma_l"], case["gamma_h"], **kw)
        want = [(c["train"], c["objective"], c["compute_fraction"]) for c in case["candidates"]]
        assert got == want, (name, case["gamma_l"], case["gamma_h"], case["machine"])


@pytest.mark.parametrize("name", ["c3_64gpu", "c4_256gpu", "t10_tiny"])
def test_partitions_vs_oracle_random_bands(name):
    import random
    rng = random.Random(31)
    orc = Oracle(problem(name))
    for _ in range(12):
        lo = rng.random() * 0.8
        hi = lo + rng.random() * 0.2
        seed = rng.randrange(1 << 40)
        fl = name == "t10_tiny" and rng.random() < 0.5
        try:
            want = oracle_partitions(orc, lo, hi, seed=seed, force_local=fl)
        except Exception:
            want = None
        if want is None:
            from paper_2511_00796_b200.engine import BandInfeasibleError
            with pytest.raises(BandInfeasibleError):
                run(name, lo, hi, seed=seed, force_local=fl)
        else:
            assert run(name, lo, hi, seed=seed, force_local=fl) == want


def test_partition_objective():
    p = problem("c3_64gpu")
    import ctypes as C

    import numpy as np
    orc = Oracle(p)
    eng = engine("c3_64gpu")
    for train in ([0, 1, 2], list(range(10, 40)), [63, 5, 17, 40]):
        ids = np.asarray(train, dtype=np.int32)
        o, f = C.c_double(), C.c_double()
        assert orc.lib.or_partition_objective(C.byref(orc.c), ids.ctypes.data_as(C.POINTER(C.c_int32)),
                                              len(ids), C.byref(o), C.byref(f)) == 0
        assert eng.partition_objective(train) == (o.value, f.value)


@pytest.mark.parametrize("csize", [1, 2, 4, 8])
@pytest.mark.parametrize("name", ["c4_256gpu", "c5_1024gpu"])
def test_restart_cluster_sizes_agree(name, csize, monkeypatch):
    """K5 runs a restart on a cluster of 1..8 CTAs (replicated state, split step scan, DSMEM
    winner exchange): every cluster size gives the C restatement's candidates. Single-band
    calls (what the schedule's later iterations make) default to 8-CTA clusters."""
    import random
    rng = random.Random(7 + csize)
    orc = Oracle(problem(name))
    monkeypatch.setenv("GPLAN_K5_CLUSTER", str(csize))
    for _ in range(3 if name == "c5_1024gpu" else 6):
        lo = 0.2 + rng.random() * 0.5
        hi = lo + 0.02 + rng.random() * 0.1
        seed = rng.randrange(1 << 40)
        want = oracle_partitions(orc, lo, hi, seed=seed)
        assert run(name, lo, hi, seed=seed) == want, (lo, hi, seed, csize)

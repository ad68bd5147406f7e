"""CPU: the host input model reproduces the reference loaders bit-for-bit."""
import numpy as np
import pytest

from common import CONFIGS, problem
from oracles import Ref


@pytest.mark.ref
@pytest.mark.parametrize("name", CONFIGS[:4])
def test_inputs_match_reference_loaders(name):
    p = problem(name)
    d = Ref(p).describe()
    cl = p.cluster
    assert [t["name"] for t in d["types"]] == cl.type_names
    for t, td in enumerate(d["types"]):
        assert td["flops"] == cl.type_flops[t]
        assert td["hbm_bandwidth"] == cl.type_hbm_bw[t]
        assert td["hbm_capacity"] == cl.type_hbm_cap[t]
        assert td["compute_efficiency"] == p.calib.compute_eff[t]
        assert td["io_efficiency"] == p.calib.io_eff[t]
    assert [tuple(x) for x in d["devices"]] == list(zip(cl.device_type.tolist(), cl.device_machine.tolist()))
    assert np.array_equal(np.asarray(d["links"]).reshape(cl.n, cl.n), cl.links)
    assert d["mean_len"] == p.workload.mean_len
    assert d["tokens_per_step"] == p.workload.tokens_per_step()
    assert d["params"]["max_concurrency"] == p.calib.max_concurrency

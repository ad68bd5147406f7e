"""CPU: the C-ABI library loads, exports every entry point include/gplan.h declares,
and refuses to run without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from common import ROOT, problem

HEADER = os.path.join(ROOT, "include", "gplan.h")
LIB = os.path.join(ROOT, "paper_2511_00796_b200", "libgplan.so")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(gp_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2511_00796_b200 import _build
        _build.build()
    return C.CDLL(LIB)


def test_exports_every_declared_symbol(lib):
    names = declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_abi_version(lib):
    assert lib.gp_abi_version() == 1


def test_no_gpu_means_loud_failure(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2511_00796_b200 import abi
    abi.declare(lib, "gp")
    c, w, k = problem("c2_16gpu").structs()
    h = C.c_void_p()
    rc = lib.gp_ctx_create(C.byref(c), C.byref(w), C.byref(k), 0, C.byref(h))
    assert rc == abi.GP_CUDA_ERROR
    assert b"no CPU fallback" in lib.gp_last_error() or b"CUDA" in lib.gp_last_error()
    from paper_2511_00796_b200.engine import Engine, EngineUnavailable
    with pytest.raises(EngineUnavailable):
        Engine(problem("c2_16gpu"))


def test_invalid_inputs_rejected_before_device(lib):
    from paper_2511_00796_b200 import abi
    abi.declare(lib, "gp")
    p = problem("c2_16gpu")
    c, w, k = p.structs()
    w.num_layers = 0
    h = C.c_void_p()
    assert lib.gp_ctx_create(C.byref(c), C.byref(w), C.byref(k), 0, C.byref(h)) == abi.GP_INVALID


def test_static_reference_build_is_not_interposed_and_the_guard_says_so():
    """The stock CMake layout links the reference STATICALLY (proj/CMakeLists.txt), so an
    LD_PRELOADed shim cannot interpose the seam: the binary keeps its own constrained_search
    & co. and silently runs on the CPU. GPLAN_REQUIRE_ENGINE=1 turns that into exit status 86
    (INTEGRATION.md); without it the static binary still produces the reference plan."""
    import json
    import os
    import subprocess

    import pytest
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cli = os.path.join(root, "oracle", "_ref", "rlsched_plan_static")
    shim = os.path.join(root, "paper_2511_00796_b200", "libgplan_shim.so")
    if not (os.path.exists(cli) and os.path.exists(shim)):
        pytest.skip("static reference CLI / shim not built (need /root/reference at build time)")
    data = os.path.join(root, "data")
    args = [cli, "--cluster", os.path.join(data, "clusters", "c1_desk_mixed.json"),
            "--workload", os.path.join(data, "workloads", "c1_desk_mixed.json"),
            "--calibration", os.path.join(data, "calibration", "c1_desk_mixed.json"), "--eta", "4"]
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        env = dict(os.environ, LD_PRELOAD=shim, GPLAN_REQUIRE_ENGINE="1")
        r = subprocess.run(args + ["--out", os.path.join(d, "a")], capture_output=True, env=env, timeout=300)
        assert r.returncode == 86, r.stderr[-2000:]
        assert b"no rlsched seam call reached the B200 engine" in r.stderr
        r = subprocess.run(args + ["--out", os.path.join(d, "b")], capture_output=True, timeout=300)
        assert r.returncode == 0
        with open(os.path.join(d, "b", "plan.json")) as f, \
                open(os.path.join(root, "tests", "golden", "desk_plan.json")) as g:
            assert json.load(f) == json.load(g)

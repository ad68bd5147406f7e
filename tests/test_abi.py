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

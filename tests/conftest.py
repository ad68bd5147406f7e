import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU and the built libgplan.so")
    config.addinivalue_line("markers", "ref: needs oracle/_ref/libref.so (reference built from /root/reference)")


def pytest_collection_modifyitems(config, items):
    from oracles import ref_available
    skip_ref = pytest.mark.skip(reason="oracle/_ref/libref.so not built here")
    for it in items:
        if "ref" in it.keywords and not ref_available():
            it.add_marker(skip_ref)

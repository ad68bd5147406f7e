"""Runs the UNMODIFIED reference schedule() with libgplan_shim.so interposed
(LD_PRELOAD set by the caller). Prints one JSON line per config."""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from common import problem  # noqa: E402
from oracles import Ref  # noqa: E402

shim = ctypes.CDLL(None).gplan_shim_calls
shim.restype = ctypes.c_longlong
for arg in sys.argv[1:]:
    name, eta = arg.split("/eta=")
    ref = Ref(problem(name))
    t = time.perf_counter()
    out = ref.schedule(eta=int(eta))
    dt = time.perf_counter() - t
    print(json.dumps({"key": arg, "plan": json.loads(out["plan_json"]), "trace": out["trace"],
                      "seconds": dt, "engine_calls": shim()}), flush=True)

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
reset = ctypes.CDLL(None).gplan_shim_reset
for arg in sys.argv[1:]:
    name, eta = arg.split("/eta=")
    ref = Ref(problem(name))
    runs = int(os.environ.get("DROPIN_RUNS", "1"))
    secs = []
    for _ in range(runs):  # first run includes CUDA runtime init; later runs: warm process,
        reset()            # fresh engine contexts (no cached MILP tables carried over)
        c0 = shim()
        t = time.perf_counter()
        out = ref.schedule(eta=int(eta))
        secs.append(time.perf_counter() - t)
    print(json.dumps({"key": arg, "plan": json.loads(out["plan_json"]), "trace": out["trace"],
                      "seconds": secs[0], "warm_seconds": secs[-1], "engine_calls": shim() - c0}),
          flush=True)

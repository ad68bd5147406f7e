#!/bin/bash
# time-to-best-plan: the unmodified reference schedule() with the engine interposed (drop-in)
# vs the reference on the host CPU. Usage: tools/time_to_plan.sh "c1_desk_mixed/eta=1 ..." [cpu]
KEYS=${1:-"c1_desk_mixed/eta=1 c2_16gpu/eta=2 c3_64gpu/eta=1"}
echo "== engine (drop-in)"
for k in $KEYS; do
  DROPIN_RUNS=2 LD_PRELOAD=$PWD/paper_2511_00796_b200/libgplan_shim.so timeout ${TTP_TIMEOUT:-900} python tests/dropin_driver.py $k | \
    python -c "import json,sys; [print(d['key'], 'cold %.3f s'%d['seconds'], 'warm %.3f s'%d['warm_seconds'], 'calls', d['engine_calls'], 'window', d['plan']['window_steps'], 'obj', max(d['plan']['costs']['train_s'], d['plan']['costs']['infer_total_s'])) for d in map(json.loads, sys.stdin)]"
done
if [ "$2" == "cpu" ]; then
  echo "== reference on host CPU"
  for k in $KEYS; do
    timeout ${TTP_TIMEOUT:-900} python - $k <<'PY'
import json, sys, time
sys.path.insert(0, "tests")
from common import problem
from oracles import Ref
name, eta = sys.argv[1].split("/eta=")
t = time.perf_counter(); out = Ref(problem(name)).schedule(eta=int(eta)); dt = time.perf_counter() - t
p = json.loads(out["plan_json"])
print(sys.argv[1], "seconds %.3f" % dt, "window", p["window_steps"])
PY
  done
fi

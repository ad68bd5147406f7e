#!/bin/bash
# 1-GPU box: schedule / drop-in / partition parity, then C5 time-to-best-plan with the phase profile
mkdir -p gpurun_out
python -m pytest tests/test_engine_schedule.py tests/test_dropin.py tests/test_engine_partition.py tests/test_engine_c4_calls.py -x -q > gpurun_out/ttp1_tests.log 2>&1; echo rc=$? >> gpurun_out/ttp1_tests.log
python tools/ttp_native.py c5_1024gpu/eta=2 c4_256gpu/eta=2 c3_64gpu/eta=1 > gpurun_out/ttp_1dev.log 2>&1
GPLAN_PROFILE=1 python tools/ttp_native.py c5_1024gpu/eta=2 > gpurun_out/ttp_1dev_prof.log 2>&1

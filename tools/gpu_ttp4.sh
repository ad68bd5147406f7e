#!/bin/bash
# 4-GPU box: schedule parity on a 4-device context (and on [0,0] with one visible GPU), then
# C5 time-to-best-plan on 1 and 4 devices
mkdir -p gpurun_out
python -m pytest tests/test_engine_schedule.py -x -q > gpurun_out/sched4_tests.log 2>&1; echo rc=$? >> gpurun_out/sched4_tests.log
CUDA_VISIBLE_DEVICES=0 python -m pytest tests/test_engine_schedule.py -x -q -k multi_device >> gpurun_out/sched4_tests.log 2>&1; echo rc=$? >> gpurun_out/sched4_tests.log
python tools/ttp_native.py c5_1024gpu/eta=2 > gpurun_out/ttp_1dev.log 2>&1
python tools/ttp_native.py c5_1024gpu/eta=2 --devices 0,1,2,3 > gpurun_out/ttp_4dev.log 2>&1
GPLAN_PROFILE=1 python tools/ttp_native.py c5_1024gpu/eta=2 --devices 0,1,2,3 > gpurun_out/ttp_4dev_prof.log 2>&1
GPLAN_PROFILE=1 python tools/ttp_native.py c5_1024gpu/eta=2 > gpurun_out/ttp_1dev_prof.log 2>&1

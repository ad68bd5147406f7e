#!/bin/bash
mkdir -p gpurun_out
for f in paper_2511_00796_b200/libgplan.so variants/libgplan_mc16.so variants/libgplan_mc64.so; do
  echo "== $f"; GPLAN_LIB=$PWD/$f python tools/k1_sizes.py
done > gpurun_out/minchunk.log 2>&1
GPLAN_LIB=$PWD/variants/libgplan_mc16.so python -m pytest tests/test_engine_train.py tests/test_engine_train_full.py -x -q > gpurun_out/mc_tests.log 2>&1; echo rc=$? >> gpurun_out/mc_tests.log

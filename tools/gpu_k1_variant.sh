#!/bin/bash
# A/B of K1-fast variant libraries (tools/build_variant.sh): K1 time alternated with the product
# library, parity of the last variant on the train tests, one ncu --set full capture of its K1.
# usage: bash tools/gpu_k1_variant.sh NAME [NAME...]   (variants/libgplan_NAME.so)
mkdir -p gpurun_out
libs=""
for n in "$@"; do libs="$libs variants/libgplan_$n.so"; done
last=variants/libgplan_${@: -1}.so
for rep in 1 2; do
  for f in paper_2511_00796_b200/libgplan.so $libs; do
    GPLAN_LIB=$PWD/$f TAG=$(basename $f .so) timeout 300 python tools/k1_time.py 2>&1 | tail -1
  done
done > gpurun_out/vt.log
GPLAN_LIB=$PWD/$last timeout 900 python -m pytest tests/test_engine_train_full.py tests/test_engine_train.py -x -q > gpurun_out/vpar.log 2>&1
GPLAN_LIB=$PWD/$last timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_layout_scan_fast -c 1 -f \
  -o gpurun_out/k1var python tools/k1_time.py > gpurun_out/ncu_var.log 2>&1

#!/bin/bash
# K1 time (tools/k1_time.py) of the product library and every variants/libgplan_*.so
cd "$(dirname "$0")/.."
for f in paper_2511_00796_b200/libgplan.so variants/libgplan_*.so; do
  GPLAN_LIB=$PWD/$f TAG="$(basename $f .so)" timeout 300 python tools/k1_time.py 2>&1 | tail -1
done

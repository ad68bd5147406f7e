#!/bin/bash
# K1 time of the product library and every variants/libgplan_*.so (tools/k1_time.py), for the
# default inner run and GPLAN_K1_INNER=$INNERS
cd "$(dirname "$0")/.."
for inner in default ${INNERS:-2}; do
  for f in paper_2511_00796_b200/libgplan.so variants/libgplan_*.so; do
    if [ "$inner" = default ]; then e=""; else e="GPLAN_K1_INNER=$inner"; fi
    env $e GPLAN_LIB=$PWD/$f TAG="$(basename $f .so) i=$inner" timeout 300 python tools/k1_time.py 2>&1 | tail -1
  done
done

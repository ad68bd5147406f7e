#!/bin/bash
# Bench each variants/libgplan_*.so (value + K1 ms only).
for f in variants/libgplan_*.so; do
  GPLAN_LIB=$PWD/$f timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-ttp 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', '%.4g'%d['value'], 'k1_ms %.2f'%d['roofline']['k1_ms_per_step'], d['winner'])"
done

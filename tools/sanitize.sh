#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_workload.py; logs in
# gpurun_out/sanitize/, one summary line per (tool, workload) on stdout.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer  # (closed on the GPU pool used in round 2: see profiles/r02/checks.md)
for tool in memcheck racecheck synccheck; do
  for w in ${WORKLOADS:-k1 k1defer k4 k5 sched}; do
    log=gpurun_out/sanitize/${tool}_${w}.log
    timeout 1500 $CS --tool $tool --print-limit 20 --target-processes all python tools/sanitize_workload.py $w > $log 2>&1
    echo "$tool $w rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $log | tail -1) $(grep -c '^ok ' $log)"
  done
done

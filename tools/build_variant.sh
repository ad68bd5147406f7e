#!/bin/bash
# build_variant.sh NAME "-DFLAG=V ..." : libgplan with extra nvcc defines -> variants/libgplan_NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=/tmp/var_$name; mkdir -p $out
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -prec-div=true -prec-sqrt=true -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include"
for s in capi train rollout partition schedule exhaustive simulate; do
  src=paper_2511_00796_b200/csrc/$s.cu
  if [ "$s" = train ]; then nvcc $F $* -c $src -o $out/$s.o; else cp paper_2511_00796_b200/_obj/$s.cu.o $out/$s.o; fi
done
mkdir -p variants
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $out/*.o -o variants/libgplan_$name.so -lcudart_static -lrt -ldl -lpthread
echo variants/libgplan_$name.so

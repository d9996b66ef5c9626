#!/bin/bash
# Bench several prebuilt library variants in one GPU call (kernel time only):
#   bash tools/gpu_bench_variants.sh TAG lib1.so lib2.so ...
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
for LIB in "$@"; do
  name=$(basename $LIB .so)
  RTK_LIBRARY=$LIB timeout 300 python bench.py --no-cpu --no-e2e --no-torch --steps 300 > $OUT/bench_$name.json 2> $OUT/bench_$name.err
done
echo done > $OUT/DONE

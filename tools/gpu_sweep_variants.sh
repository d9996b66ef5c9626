#!/bin/bash
# Sweep a subset of shapes for several library variants (kernel time only):
#   bash tools/gpu_sweep_variants.sh TAG "M:k,M:k" lib1.so lib2.so ...
TAG=$1; SHAPES=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
for LIB in "$@"; do
  name=$(basename $LIB .so)
  RTK_LIBRARY=$LIB timeout 600 python tools/sweep_bench.py --shapes "$SHAPES" --no-extra --no-torch --steps 30 > $OUT/sweep_$name.log 2>&1
done
echo done > $OUT/DONE

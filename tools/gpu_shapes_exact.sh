#!/bin/bash
# Kernel time of library variants over several shapes (exact mode, or
# MODE=early):   bash tools/gpu_shapes_exact.sh TAG "lib1 lib2" "N:M:k ..."
TAG=$1; LIBS=$2; SHAPES=$3; MODE=${MODE:-exact}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for SH in $SHAPES; do
  for LIB in $LIBS; do
    B=$(basename $LIB .so)
    RTK_LIBRARY=$LIB timeout 300 python bench.py --mode $MODE --only-mode --no-torch --no-cpu --no-e2e --no-c5 \
      --steps 100 --warmup 5 --shape $SH > $OUT/b_${B}_$(echo $SH | tr ':' '_')_$MODE.json 2>> $OUT/err.log
  done
done
echo done > $OUT/DONE

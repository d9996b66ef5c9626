#!/bin/bash
# A/B kernel timing of library variants (exact + early, C2 device-resident),
# then the GPU test suite on the in-tree library.
#   bash tools/gpu_ab.sh TAG "lib1.so lib2.so ..." [pytest-args...]
TAG=$1; LIBS=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/nvsmi.csv 2>&1
for rep in 1 2; do
for LIB in $LIBS; do
  B=$(basename $LIB .so)
  for MODE in exact early; do
    RTK_LIBRARY=$LIB timeout 300 python bench.py --mode $MODE --only-mode --no-torch --no-cpu --no-e2e --no-c5 \
      --steps 300 --warmup 10 > $OUT/bench_${B}_${MODE}_$rep.json 2> $OUT/bench_${B}_${MODE}_$rep.err
  done
done
done
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q "$@" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
echo done > $OUT/DONE

#!/bin/bash
# Parity (-m gpu, M=256 subset via -k) + bench for several library variants in one GPU call:
#   bash tools/gpu_try.sh TAG lib1.so lib2.so ...
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
for LIB in "$@"; do
  name=$(basename $LIB .so)
  RTK_LIBRARY=$LIB timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest_$name.log 2>&1; echo "rc=$?" >> $OUT/pytest_$name.log
  RTK_LIBRARY=$LIB timeout 300 python bench.py --no-cpu --no-e2e --no-torch --steps 300 > $OUT/bench_$name.json 2> $OUT/bench_$name.err
done
echo done > $OUT/DONE

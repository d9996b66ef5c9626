#!/bin/bash
# Parity tests + bench for one prebuilt library variant: bash tools/gpu_variant.sh TAG LIB [ncu]
TAG=$1; LIB=$2
OUT=gpurun_out/$TAG
mkdir -p $OUT
export RTK_LIBRARY=$LIB
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python bench.py --no-cpu --no-e2e --no-torch --steps 300 > $OUT/bench.json 2> $OUT/bench.err
if [ "${3:-}" = "ncu" ]; then
for MODE in ${4:-exact early}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rowtopk_kernel|pair_kernel" -s 3 -c 1 \
    -o /tmp/prof_$MODE python bench.py --mode $MODE --steps 2 --warmup 3 --no-cpu --no-e2e --only-mode --no-torch > $OUT/ncu_full_$MODE.log 2>&1
ncu -i /tmp/prof_$MODE.ncu-rep --page raw --csv > $OUT/prof_${MODE}_raw.csv 2>/dev/null
ncu -i /tmp/prof_$MODE.ncu-rep --page source --csv --print-source sass > $OUT/prof_${MODE}_src.csv 2>/dev/null
ncu -i /tmp/prof_$MODE.ncu-rep --page details > $OUT/prof_${MODE}_details.txt 2>/dev/null
done
fi
echo done > $OUT/DONE

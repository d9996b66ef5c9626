#!/bin/bash
# ncu --set full capture of one rowtopk launch per mode for a library variant; exports CSV/text.
#   bash tools/gpu_ncu_variant.sh TAG LIB [modes]
TAG=$1; LIB=$2; MODES=${3:-"exact early"}; SHAPE=${4:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export RTK_LIBRARY=$LIB
for MODE in $MODES; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rowtopk -s 3 -c 1 -f \
    -o /tmp/prof_$MODE python bench.py --mode $MODE --steps 2 --warmup 3 --no-cpu --no-e2e --only-mode --no-torch ${SHAPE:+--shape $SHAPE} > $OUT/ncu_full_$MODE.log 2>&1
ncu -i /tmp/prof_$MODE.ncu-rep --page raw --csv > $OUT/prof_${MODE}_raw.csv 2>/dev/null
ncu -i /tmp/prof_$MODE.ncu-rep --page source --csv --print-source sass > $OUT/prof_${MODE}_src.csv 2>/dev/null
ncu -i /tmp/prof_$MODE.ncu-rep --page details > $OUT/prof_${MODE}_details.txt 2>/dev/null
done
echo done > $OUT/DONE

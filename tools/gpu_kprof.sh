#!/bin/bash
# Kernel iteration on the GPU box: bench (exact + early, device-resident C2)
# for each library given, then one ncu --set full capture of the hot kernel
# per mode for the first library (raw / source / details exported as text).
#   bash tools/gpu_kprof.sh TAG "LIB1 LIB2 ..." [modes] [N:M:k]
TAG=$1; LIBS=$2; MODES=${3:-"exact early"}; SHAPE=${4:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for LIB in $LIBS; do
  B=$(basename $LIB .so)
  for MODE in $MODES; do
    RTK_LIBRARY=$LIB timeout 300 python bench.py --mode $MODE --only-mode --no-torch --no-cpu --no-e2e \
      --steps 200 --warmup 10 ${SHAPE:+--shape $SHAPE} > $OUT/bench_${B}_$MODE.json 2> $OUT/bench_${B}_$MODE.err
  done
done
FIRST=$(echo $LIBS | awk '{print $1}')
if [ "${NCU:-1}" = "1" ]; then
for MODE in $MODES; do
  RTK_LIBRARY=$FIRST timeout 600 ncu --set full --clock-control none --import-source on -k regex:rowtopk -s 3 -c 1 -f \
      -o /tmp/kprof_$MODE python bench.py --mode $MODE --steps 2 --warmup 3 --no-cpu --no-e2e --only-mode --no-torch \
      ${SHAPE:+--shape $SHAPE} > $OUT/ncu_$MODE.log 2>&1
  ncu -i /tmp/kprof_$MODE.ncu-rep --page raw --csv > $OUT/prof_${MODE}_raw.csv 2>/dev/null
  ncu -i /tmp/kprof_$MODE.ncu-rep --page source --csv --print-source sass > $OUT/prof_${MODE}_src.csv 2>/dev/null
  ncu -i /tmp/kprof_$MODE.ncu-rep --page details > $OUT/prof_${MODE}_details.txt 2>/dev/null
done
fi
echo done > $OUT/DONE

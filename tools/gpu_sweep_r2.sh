#!/bin/bash
# Clock-recorded sweep (BASELINE configs[2..3] through bench.py; C5 is a leg of the default bench line) + ncu captures
# of the M=128 and M=768 kernels.   bash tools/gpu_sweep_r2.sh TAG
TAG=${1:-sweep}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/nvsmi.csv 2>&1
timeout 1200 python bench.py --sweep --steps 50 --warmup 5 > $OUT/sweep.jsonl 2> $OUT/sweep.err
if [ "${NCU:-1}" = "1" ]; then
for SH in 1048576:128:32 1048576:768:64; do
  for MODE in exact early; do
    T=$(echo $SH | tr ':' '_')_$MODE
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:rowtopk -s 3 -c 1 -f \
        -o /tmp/ncu_$T python bench.py --mode $MODE --steps 2 --warmup 3 --no-cpu --no-e2e --only-mode --no-torch \
        --shape $SH > $OUT/ncu_$T.log 2>&1
    ncu -i /tmp/ncu_$T.ncu-rep --page raw --csv > $OUT/prof_${T}_raw.csv 2>/dev/null
    ncu -i /tmp/ncu_$T.ncu-rep --page source --csv --print-source sass > $OUT/prof_${T}_src.csv 2>/dev/null
    ncu -i /tmp/ncu_$T.ncu-rep --page details > $OUT/prof_${T}_details.txt 2>/dev/null
  done
done
fi
echo done > $OUT/DONE

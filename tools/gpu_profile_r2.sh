#!/bin/bash
# Round-2 evidence on one GPU: the default bench line (C2 + e2e + CPU baseline
# + C5 leg), the early-stop line, the reference arm, the ncu launch list of the
# default bench command, ncu --set full captures (C2 exact/early, C5 shape
# exact/early, M=1024 exact), the clock-recorded sweep, MaxK bench, GPU tests
# and smoke.   bash tools/gpu_profile_r2.sh TAG
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/nvsmi.csv 2>&1
timeout 900 python bench.py > $OUT/bench_exact.json 2> $OUT/bench_exact.err
timeout 600 python bench.py --mode early --no-c5 > $OUT/bench_early.json 2> $OUT/bench_early.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 120 python bench.py --gpus 2 > $OUT/bench_gpus2.out 2>&1; echo "rc=$?" >> $OUT/bench_gpus2.out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-c5 > $OUT/ncu_launch.log 2>&1
run_full() {  # name mode shape
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:rowtopk -s 3 -c 1 -f -o /tmp/prof_$1 \
      python bench.py --mode $2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-c5 --only-mode --no-torch ${3:+--shape $3} > $OUT/ncu_full_$1.log 2>&1
  ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > $OUT/prof_$1_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$1.ncu-rep --page details > $OUT/prof_$1_details.txt 2>/dev/null
  ncu -i /tmp/prof_$1.ncu-rep --page source --csv --print-source sass > $OUT/prof_$1_src.csv 2>/dev/null
}
run_full c2_exact exact
run_full c2_early early
run_full m512_exact exact 1048576:512:64
run_full m512_early early 1048576:512:64
run_full m1024_exact exact 1048576:1024:64
timeout 1200 python bench.py --sweep --steps 50 --warmup 5 > $OUT/sweep.jsonl 2> $OUT/sweep.err
timeout 600 python tools/maxk_bench.py > $OUT/maxk_bench.json 2> $OUT/maxk_bench.err
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
echo done > $OUT/DONE

#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + one full capture.
# Usage (under gpurun): bash tools/gpu_round.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --mode early > $OUT/bench_early.json 2> $OUT/bench_early.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rowtopk_kernel -c 40 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rowtopk_kernel -s 3 -c 1 \
    -o $OUT/prof_exact python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_full_exact.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rowtopk_kernel -s 3 -c 1 \
    -o $OUT/prof_early python bench.py --mode early --steps 2 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_full_early.log 2>&1
echo done > $OUT/DONE

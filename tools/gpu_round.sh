#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + one full capture per mode.
# .ncu-rep files stay in /tmp on the box (gpurun copies back <= 64 MiB); CSV/text exports come back.
# Usage (under gpurun): bash tools/gpu_round.sh [tag] [bench-args...]
TAG=${1:-r1}
shift || true
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py "$@" > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --mode early "$@" > $OUT/bench_early.json 2> $OUT/bench_early.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_launch.log 2>&1
for MODE in exact early; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rowtopk -s 3 -c 1 \
    -o /tmp/prof_$MODE -f python bench.py --mode $MODE --only-mode --no-torch --steps 2 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_full_$MODE.log 2>&1
ncu -i /tmp/prof_$MODE.ncu-rep --page raw --csv > $OUT/prof_${MODE}_raw.csv 2>/dev/null
ncu -i /tmp/prof_$MODE.ncu-rep --page details > $OUT/prof_${MODE}_details.txt 2>/dev/null
ncu -i /tmp/prof_$MODE.ncu-rep --page source --csv --print-source sass > $OUT/prof_${MODE}_src.csv 2>/dev/null
done
echo done > $OUT/DONE

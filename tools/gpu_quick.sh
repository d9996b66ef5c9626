#!/bin/bash
# Quick GPU iteration: parity tests + bench (both modes) + one ncu source capture.
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python bench.py --no-cpu --no-e2e > $OUT/bench.json 2> $OUT/bench.err
if [ "${2:-}" = "ncu" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rowtopk_kernel -s 3 -c 1 \
    -o $OUT/prof_exact python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --only-mode --no-torch > $OUT/ncu_full_exact.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rowtopk_kernel -s 3 -c 1 \
    -o $OUT/prof_early python bench.py --mode early --steps 2 --warmup 3 --no-cpu --no-e2e --only-mode --no-torch > $OUT/ncu_full_early.log 2>&1
fi
echo done > $OUT/DONE

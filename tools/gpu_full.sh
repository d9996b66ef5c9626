#!/bin/bash
# Full-library GPU check: parity tests, smoke, default bench (both modes), sweep.
TAG=${1:-full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python tools/sweep_bench.py --out $OUT/sweep.json > $OUT/sweep.log 2>&1
echo done > $OUT/DONE

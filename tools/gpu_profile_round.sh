#!/bin/bash
# Round evidence on one GPU: bench lines (both modes + reference arm), the ncu
# launch list of the default bench command, and ncu --set full captures of the
# hot kernel at C2 (exact, early) plus the long-row kernel at M=512/1024.
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python bench.py > $OUT/bench_exact.json 2> $OUT/bench_exact.err
timeout 600 python bench.py --mode early > $OUT/bench_early.json 2> $OUT/bench_early.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_launch.log 2>&1
run_full() {  # name mode shape
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:rowtopk -s 3 -c 1 -f -o /tmp/prof_$1 \
      python bench.py --mode $2 --steps 2 --warmup 3 --no-cpu --no-e2e --only-mode --no-torch ${3:+--shape $3} > $OUT/ncu_full_$1.log 2>&1
  ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > $OUT/prof_$1_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$1.ncu-rep --page details > $OUT/prof_$1_details.txt 2>/dev/null
  ncu -i /tmp/prof_$1.ncu-rep --page source --csv --print-source sass > $OUT/prof_$1_src.csv 2>/dev/null
}
run_full c2_exact exact
run_full c2_early early
run_full m1024_exact exact 1048576:1024:64
run_full m1024_early early 1048576:1024:64
run_full m512_early early 1048576:512:64
run_full m2048_exact exact 524288:2048:64
run_full m2048_early early 524288:2048:64
run_full m8192_exact exact 131072:8192:128
timeout 900 python tools/sweep_bench.py --out $OUT/sweep.json > $OUT/sweep.log 2>&1
timeout 600 python tools/x16_bench.py > $OUT/x16_bench.jsonl 2> $OUT/x16.err
timeout 600 python tools/maxk_bench.py > $OUT/maxk_bench.json 2> $OUT/maxk_bench.err
timeout 900 python tools/sweep_bench.py --shapes "1100:32,1536:64,2048:64,2500:64,3072:128,4000:64,4096:128,4500:64,6144:128,8192:128" --no-extra --no-torch --steps 30 > $OUT/sweep_long.log 2>&1
timeout 600 python tools/file_bench.py /dev/shm > $OUT/file_bench_tmpfs.json 2> $OUT/file_bench.err
timeout 300 python tools/pcie_probe.py > $OUT/pcie_probe.json 2>&1
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
echo done > $OUT/DONE

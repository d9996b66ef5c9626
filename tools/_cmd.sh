mkdir -p gpurun_out/sw3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/sw3/pytest.log 2>&1
python tools/sweep_bench.py --out gpurun_out/sw3/sweep.json > gpurun_out/sw3/log.txt 2>&1

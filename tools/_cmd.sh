mkdir -p gpurun_out/mi
for mi in 1 2 4 8 16; do
python bench.py --mode early --max-iter $mi --only-mode --no-cpu --no-e2e --no-torch --steps 300 > gpurun_out/mi/mi_$mi.json 2>/dev/null
done
for mi in 1 4 16; do
RTK_LIBRARY=build_variants/librtk_d3_512.so python bench.py --mode early --max-iter $mi --only-mode --no-cpu --no-e2e --no-torch --steps 300 > gpurun_out/mi/mi512_$mi.json 2>/dev/null
done

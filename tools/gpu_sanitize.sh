#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_probe.py
OUT=gpurun_out/${1:-sanitize}; mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  echo "## $tool" >> $OUT/sanitizer.txt
  timeout 2400 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py >> $OUT/sanitizer.txt 2>&1
done
echo done > $OUT/DONE

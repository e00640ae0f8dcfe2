#!/bin/bash
OUT=gpurun_out/${1:-trace2}
mkdir -p $OUT
for cfg in "conv3x3 512 512 4 128" "conv3x3 256 256 8 128" "conv3x3 128 128 16 128" "conv3x3_s2 64 128 16 128" "sep_shared 64 64 32 128"; do
  echo "### $cfg" >> $OUT/trace.txt
  SYNO_TC_TRACE=1 timeout 120 python scripts/gemm_probe.py $cfg 1 2>&1 | grep -A1 "tc trace" | head -12 >> $OUT/trace.txt
done

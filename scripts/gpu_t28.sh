#!/bin/bash
OUT=gpurun_out/${1:-t28}
mkdir -p $OUT
for shape in "conv3x3 64 64 32 128" "conv3x3 128 128 16 128" "conv3x3 256 256 8 128"; do
  for dbg in 0 1 13 269 271; do
    echo "### $shape dbg=$dbg" >> $OUT/cmp.txt
    SYNO_TC_DEBUG=$dbg timeout 120 python scripts/gemm_probe.py $shape 10 2>&1 | grep -E "tc_gemm_fwd" >> $OUT/cmp.txt
  done
done

#!/bin/bash
# which operand loads bound the GEMM: skip A (4) / B (8) / both (12) loads, MMA only (13)
OUT=gpurun_out/${1:-t26}
mkdir -p $OUT
for shape in "conv3x3 64 64 32 128" "conv3x3 128 128 16 128" "conv3x3 256 256 8 128"; do
  for small in 1 0; do
    for dbg in 0 4 8 12 13; do
      echo "### $shape small=$small dbg=$dbg" >> $OUT/cmp.txt
      SYNO_TC_SMALL=$small SYNO_TC_DEBUG=$dbg timeout 120 python scripts/gemm_probe.py $shape 10 2>&1 | grep -E "tc_gemm_(fwd|wgrad)" >> $OUT/cmp.txt
    done
  done
done

#!/bin/bash
OUT=gpurun_out/${1:-t24}
mkdir -p $OUT
export SYNO_TC_SMALL=0
for dbg in 0 128 13 141; do
  echo "### dbg=$dbg" >> $OUT/trace.txt
  SYNO_TC_DEBUG=$dbg SYNO_TC_TRACE=1 timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 1 2>&1 | grep -A1 "mode=0" | head -2 >> $OUT/trace.txt
  SYNO_TC_DEBUG=$dbg timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 10 2>&1 | grep tc_gemm >> $OUT/trace.txt
done

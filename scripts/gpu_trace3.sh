#!/bin/bash
OUT=gpurun_out/${1:-trace3}
mkdir -p $OUT
for dbg in 0 4 8 12; do
  echo "### 256@8 dbg=$dbg" >> $OUT/trace.txt
  SYNO_TC_DEBUG=$dbg SYNO_TC_TRACE=1 timeout 120 python scripts/gemm_probe.py conv3x3 256 256 8 128 1 2>&1 | grep -A1 "mode=0" | head -2 >> $OUT/trace.txt
  SYNO_TC_DEBUG=$dbg SYNO_NO_PDL=1 SYNO_TC_TRACE=1 timeout 120 python scripts/gemm_probe.py conv3x3 256 256 8 128 1 2>&1 | grep -A1 "mode=0" | head -2 >> $OUT/trace.txt
done

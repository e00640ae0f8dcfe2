#!/bin/bash
OUT=gpurun_out/${1:-t29}
mkdir -p $OUT
for dbg in 271 269; do
  SYNO_TC_DEBUG=$dbg SYNO_TC_TRACE=$PWD/$OUT/d$dbg.txt timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 1 > /dev/null 2>&1
done

#!/bin/bash
OUT=gpurun_out/${1:-t25}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > $OUT/tc.log 2>&1
SYNO_TC_LOG=1 timeout 300 python bench.py --no-cpu-baseline --steps 1 --warmup 1 --no-graph > $OUT/log_r18.txt 2>&1
for dbg in 0 13; do
  echo "### cfg1 dbg=$dbg" >> $OUT/trace.txt
  SYNO_TC_DEBUG=$dbg SYNO_TC_TRACE=1 timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 1 2>&1 | grep -A1 "mode=0" | head -2 >> $OUT/trace.txt
  SYNO_TC_DEBUG=$dbg timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 10 2>&1 | grep tc_gemm >> $OUT/trace.txt
done

#!/bin/bash
# GEMM component probe: per-class times with parts of the tcgen05 kernel disabled.
OUT=gpurun_out/${1:-probe}
mkdir -p $OUT
for cfg in "conv3x3 64 64 32 128" "sep_shared 64 64 32 128" "conv3x3 128 128 16 128" "conv3x3 256 256 8 128" \
           "conv3x3 512 512 4 128" "conv3x3_s2 64 128 16 128" "conv3x3 64 64 56 256" "qkv 0 0 0 16"; do
  for dbg in 0 1 2 12 13; do
    echo "### $cfg dbg=$dbg"
    SYNO_TC_DEBUG=$dbg timeout 120 python scripts/gemm_probe.py $cfg 10 2>&1 | grep -E "tc_gemm|GFLOP|Error|error"
  done
done > $OUT/probe.txt 2>&1
timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 10 > $OUT/all_classes.txt 2>&1
SYNO_TC_TRACE=1 timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 1 > $OUT/trace.txt 2>&1

#!/bin/bash
# Instruction-fetch experiment: each chain-rule launch repeated at once (SYNO_TC_CHAIN_TWICE, timing only).
OUT=gpurun_out/r02_twice
mkdir -p $OUT
for L in "sep_shared 64 64 32 128" "conv3x3 64 64 32 128" "sep_shared 512 512 4 128" "conv3x3 512 512 4 128"; do
  n=${L// /_}
  SYNO_TC_CHAIN_TWICE=1 timeout 300 python scripts/gemm_probe.py $L > $OUT/probe_$n.log 2>&1
  SYNO_TC_CHAIN_TWICE=1 SYNO_TC_NO_CHAIN_V4=1 timeout 300 python scripts/gemm_probe.py $L > $OUT/probe_old_$n.log 2>&1
done

#!/bin/bash
# Vectorised chain rule (chain_v4) A/B against the previous kernels (SYNO_TC_NO_CHAIN_V4) + full GPU suite.
OUT=gpurun_out/${1:-r02_v4}
mkdir -p $OUT
for L in "sep_shared 64 64 32 128" "sep_shared 128 128 16 128" "sep_shared 512 512 4 128" "conv3x3 64 64 32 128" "conv3x3 512 512 4 128"; do
  n=${L// /_}
  timeout 300 python scripts/gemm_probe.py $L > $OUT/probe_$n.log 2>&1
  SYNO_TC_NO_CHAIN_V4=1 timeout 300 python scripts/gemm_probe.py $L > $OUT/probe_old_$n.log 2>&1
done
for i in 1 2; do
  timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_r18_$i.log 2>&1
  SYNO_TC_NO_CHAIN_V4=1 timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_r18_old_$i.log 2>&1
done
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log

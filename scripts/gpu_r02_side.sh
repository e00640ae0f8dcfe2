#!/bin/bash
# sep_shared chain: fused side output vs two launches (SYNO_TC_NO_SIDE_CHAIN); full GPU suite.
OUT=gpurun_out/r02_side
mkdir -p $OUT
for L in "sep_shared 64 64 32 128" "sep_shared 128 128 16 128" "sep_shared 512 512 4 128"; do
  n=${L// /_}
  timeout 300 python scripts/gemm_probe.py $L > $OUT/probe_$n.log 2>&1
  SYNO_TC_NO_SIDE_CHAIN=1 timeout 300 python scripts/gemm_probe.py $L > $OUT/probe_noside_$n.log 2>&1
done
timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_r18.log 2>&1
SYNO_TC_NO_SIDE_CHAIN=1 timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_r18_noside.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log

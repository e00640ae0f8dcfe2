#!/bin/bash
# BN = 128 GEMMs in CTA pairs (SYNO_TC_PAIR128=1) vs two CTAs per SM: parity + timing.
OUT=gpurun_out/r02_pair128
mkdir -p $OUT
SYNO_TC_PAIR128=1 timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_bench_shapes.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for c in "pair:SYNO_TC_PAIR128=1" "base:"; do
  n=${c%%:*}; e=${c#*:}
  for args in "conv3x3 128 128 16 128" "conv3x3_s2 64 128 16 128" "sep_shared 128 128 16 128" "conv3x3 128 128 28 256"; do
    echo "## $n $args" >> $OUT/ab.txt
    env $e timeout 120 python scripts/gemm_probe.py $args 10 2>&1 | grep tc_gemm >> $OUT/ab.txt
  done
  env $e timeout 300 python bench.py --no-cpu-baseline > $OUT/bench18_$n.log 2>&1
  env $e timeout 300 python bench.py --workload resnet34 --no-cpu-baseline > $OUT/bench34_$n.log 2>&1
done

#!/bin/bash
# Flat-pixel pack blocks (14 x 14 maps: 4-wide loads) vs row blocks: parity + ResNet-34 timing.
OUT=gpurun_out/r02_flat
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_bench_shapes.py tests/test_gpu_parity.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for c in "flat:" "rows:SYNO_TC_NO_FLAT_PACK=1"; do
  n=${c%%:*}; e=${c#*:}
  env $e timeout 120 python scripts/gemm_probe.py conv3x3 256 256 14 256 10 > $OUT/probe14_$n.txt 2>&1
  env $e timeout 300 python bench.py --workload resnet34 --no-cpu-baseline > $OUT/bench34_$n.log 2>&1
done

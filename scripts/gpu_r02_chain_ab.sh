#!/bin/bash
# Chain-rule kernel A/B: per-layer class times and the ResNet-18 step, chain_win vs chain_nc for
# single-weight convolutions (SYNO_TC_NO_CHAIN_WIN), then the chain-touching GPU tests.
OUT=gpurun_out/r02_chain_ab
mkdir -p $OUT
for L in "sep_shared 64 64 32 128" "sep_shared 512 512 4 128" "conv3x3 64 64 32 128" "conv3x3 512 512 4 128" "conv3x3 256 256 8 128"; do
  n=${L// /_}
  timeout 300 python scripts/gemm_probe.py $L > $OUT/probe_$n.log 2>&1
  SYNO_TC_NO_CHAIN_WIN=1 timeout 300 python scripts/gemm_probe.py $L > $OUT/probe_nowin_$n.log 2>&1
done
for i in 1 2; do
  timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_r18_$i.log 2>&1
  SYNO_TC_NO_CHAIN_WIN=1 timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_r18_nowin_$i.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_bench_shapes.py tests/test_gpu_tc.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log

#!/bin/bash
# chain_v4 with the last block's partial loads batched: per-launch times, ResNet-18 A/B, full GPU suite.
OUT=gpurun_out/${1:-r02_v4d}
mkdir -p $OUT
for L in "sep_shared 64 64 32 128" "sep_shared 128 128 16 128" "sep_shared 512 512 4 128"; do
  n=${L// /_}
  for cfg in "base:" "old:SYNO_TC_NO_CHAIN_V4=1" "wred:SYNO_TC_V4_WRED=1" "nowred:SYNO_TC_V4_WRED=0"; do
    tag=${cfg%%:*}; envs=${cfg#*:}
    env $envs timeout 300 python scripts/gemm_probe.py $L > $OUT/probe_${tag}_$n.log 2>&1
  done
done
for i in 1 2; do
  timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_base_$i.log 2>&1
  SYNO_TC_V4_WRED=0 timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_wred_$i.log 2>&1
done
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log

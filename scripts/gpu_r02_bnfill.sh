#!/bin/bash
# Tile-count-aware BN (SYNO_TC_BN_FILL) A/B on every layer workload, then the full GPU suite.
OUT=gpurun_out/${1:-r02_bnfill}
mkdir -p $OUT
for i in 1 2; do
  for cfg in "base:" "old:SYNO_TC_BN_FILL=0 SYNO_TC_WG_BN_FILL=0" "nowg:SYNO_TC_WG_BN_FILL=0"; do
    tag=${cfg%%:*}; envs=${cfg#*:}
    env $envs timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_r18_${tag}_$i.log 2>&1
  done
done
for w in resnet34 qkv cfg1; do
  for cfg in "base:" "old:SYNO_TC_BN_FILL=0 SYNO_TC_WG_BN_FILL=0"; do
    tag=${cfg%%:*}; envs=${cfg#*:}
    env $envs timeout 600 python bench.py --workload $w --no-cpu-baseline > $OUT/bench_${w}_${tag}.log 2>&1
  done
done
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log

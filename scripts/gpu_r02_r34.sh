#!/bin/bash
# ResNet-34 tiling switches (per-layer breakdown in each line).
OUT=gpurun_out/r02_r34
mkdir -p $OUT
for cfg in "base:" "small0:SYNO_TC_SMALL=0" "g1:SYNO_TC_G=1" "max128:SYNO_TC_MAXBN=128" "nors:SYNO_TC_NO_RSPLIT=1"; do
  tag=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 600 python bench.py --workload resnet34 --no-cpu-baseline > $OUT/bench_${tag}.log 2>&1
done

#!/bin/bash
# Tiling A/B on the ResNet-18 step: BN cap, channel split off, both (layer-level switches).
OUT=gpurun_out/r02_tiling
mkdir -p $OUT
for i in 1 2; do
  for cfg in "base:" "bn128:SYNO_TC_MAXBN=128" "nors:SYNO_TC_NO_RSPLIT=1" "bn128nors:SYNO_TC_MAXBN=128 SYNO_TC_NO_RSPLIT=1" "waves2:SYNO_TC_WG_WAVES=2"; do
    tag=${cfg%%:*}; envs=${cfg#*:}
    env $envs timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_${tag}_$i.log 2>&1
  done
done

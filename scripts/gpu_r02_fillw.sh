#!/bin/bash
# Tile-count rule threshold: 1 vs 2 vs 3 waves of 256-wide tiles (SYNO_TC_BN_FILL_WAVES).
OUT=gpurun_out/r02_fillw
mkdir -p $OUT
for w in resnet18 resnet34; do
  for fw in 1 2 3; do
    SYNO_TC_BN_FILL_WAVES=$fw timeout 600 python bench.py --workload $w --no-others --no-cpu-baseline > $OUT/bench_${w}_w$fw.log 2>&1
  done
done

#!/bin/bash
OUT=gpurun_out/r02_carve
mkdir -p $OUT
for c in 1 0 1 0; do
  SYNO_CARVEOUT=$c timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_c$c.log 2>&1
  python -c "import json;d=[json.loads(l) for l in open('$OUT/bench_c$c.log') if l.startswith('{')][0];print('carveout=$c', d['ms_per_step'], d['value'])" >> $OUT/summary.txt
done
for c in 1 0; do
  for args in "conv3x3 64 64 32 128" "shortcut_s2 64 128 16 128" "conv3x3 3 64 32 128"; do
    echo "## c=$c $args" >> $OUT/summary.txt
    SYNO_CARVEOUT=$c timeout 120 python scripts/gemm_probe.py $args 10 2>&1 | tail -n +2 >> $OUT/summary.txt
  done
done

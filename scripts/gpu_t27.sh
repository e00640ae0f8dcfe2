#!/bin/bash
OUT=gpurun_out/${1:-t27}
mkdir -p $OUT
for shape in "conv3x3 64 64 32 128" "conv3x3 128 128 16 128"; do
  for dbg in 0 13; do
    tag=$(echo $shape | tr ' ' '_')_d$dbg
    SYNO_TC_DEBUG=$dbg SYNO_TC_TRACE=$PWD/$OUT/$tag.txt timeout 120 python scripts/gemm_probe.py $shape 1 > /dev/null 2>&1
  done
done
ls -la $OUT

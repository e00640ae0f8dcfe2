#!/bin/bash
# In-graph attribution of the ResNet-18 step: time with each kernel class suppressed.
OUT=gpurun_out/${1:-attrib}
mkdir -p $OUT
for sk in "" pack fold chain cast zero gemm "pack,fold,chain,cast,zero"; do
  echo "### skip=$sk" >> $OUT/attrib.txt
  SYNO_SKIP=$sk timeout 300 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])" >> $OUT/attrib.txt
done

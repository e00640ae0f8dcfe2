#!/bin/bash
OUT=gpurun_out/${1:-t23}
mkdir -p $OUT
for v in 256 128; do
  export SYNO_TC_MAXBN=$v
  echo "### maxbn=$v" >> $OUT/cmp.txt
  for cfg in "conv3x3 256 256 8 128" "conv3x3 512 512 4 128" "qkv 0 0 0 16"; do
    timeout 120 python scripts/gemm_probe.py $cfg 10 2>&1 | grep -E "tc_gemm" >> $OUT/cmp.txt
  done
  echo "r18 $(timeout 300 python bench.py --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/cmp.txt
  echo "r34 $(timeout 300 python bench.py --workload resnet34 --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/cmp.txt
  echo "qkv $(timeout 300 python bench.py --workload qkv --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/cmp.txt
done

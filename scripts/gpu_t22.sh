#!/bin/bash
OUT=gpurun_out/${1:-t22}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for v in 1 0; do
  export SYNO_TC_SMALL=$v
  echo "### small=$v" >> $OUT/cmp.txt
  for cfg in "conv3x3 64 64 32 128" "conv3x3 128 128 16 128"; do
    timeout 120 python scripts/gemm_probe.py $cfg 10 2>&1 | grep -E "tc_gemm" >> $OUT/cmp.txt
  done
  echo "r18 $(timeout 300 python bench.py --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/cmp.txt
  echo "r34 $(timeout 300 python bench.py --workload resnet34 --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/cmp.txt
done

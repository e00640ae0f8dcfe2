#!/bin/bash
OUT=gpurun_out/${1:-t32}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > $OUT/tc.log 2>&1
for v in 0 1; do
  if [ $v = 1 ]; then export SYNO_TC_NO_BRES=1; fi
  echo "### nobres=$v" >> $OUT/cmp.txt
  for shape in "conv3x3 64 64 32 128" "conv3x3 3 64 32 128" "conv3x3 128 128 16 128"; do
    timeout 120 python scripts/gemm_probe.py $shape 10 2>&1 | grep -E "tc_gemm_(fwd|dgrad|wgrad)" >> $OUT/cmp.txt
  done
  echo "r18 $(timeout 300 python bench.py --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/cmp.txt
  echo "r34 $(timeout 300 python bench.py --workload resnet34 --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/cmp.txt
done

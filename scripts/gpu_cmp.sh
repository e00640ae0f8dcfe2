#!/bin/bash
# Quick A/B evidence: tc parity tests, per-layer probes, step times of the three layer benches.
OUT=gpurun_out/${1:-cmp}
mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2 > $OUT/tc.log
for shape in "qkv 768 2304 1024 16" "conv3x3 64 64 32 128" "conv3x3 128 128 16 128" "conv3x3 256 256 14 256"; do
  echo "## $shape" >> $OUT/probe.txt
  timeout 120 python scripts/gemm_probe.py $shape 10 2>&1 | grep -E "tc_gemm|pack|chain|fold" >> $OUT/probe.txt
done
for wl in resnet18 resnet34 qkv; do
  echo "$wl $(timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'], d['roofline']['frac'])")" >> $OUT/bench.txt
done
cat $OUT/tc.log $OUT/probe.txt $OUT/bench.txt

#!/bin/bash
OUT=gpurun_out/${1:-t8}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_resnet18.log 2>&1
timeout 600 python bench.py --workload resnet34 --steps 5 --no-cpu-baseline > $OUT/bench_resnet34.log 2>&1
timeout 600 python bench.py --workload cfg1 --no-cpu-baseline > $OUT/bench_cfg1.log 2>&1
timeout 600 python bench.py --workload qkv --no-cpu-baseline > $OUT/bench_qkv.log 2>&1
for cfg in "conv3x3 64 64 32 128" "sep_shared 64 64 32 128" "conv3x3 256 256 8 128" "conv3x3 512 512 4 128"; do
  timeout 120 python scripts/gemm_probe.py $cfg 10 >> $OUT/probe.txt 2>&1
done

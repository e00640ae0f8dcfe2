#!/bin/bash
# GPU test pass + probe.  usage: bash scripts/gpu_test.sh <tag>
OUT=gpurun_out/${1:-t}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python scripts/sweep_fail.py 8 170 518 732 828 > $OUT/sweep_fail.txt 2>&1
for cfg in "conv3x3 64 64 32 128" "sep_shared 64 64 32 128" "conv3x3 128 128 16 128" "conv3x3 256 256 8 128" \
           "conv3x3 512 512 4 128" "conv3x3_s2 64 128 16 128" "qkv 0 0 0 16"; do
  timeout 120 python scripts/gemm_probe.py $cfg 10 >> $OUT/probe.txt 2>&1
done
timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 8 10 float32 >> $OUT/probe.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_resnet18.log 2>&1
timeout 600 python bench.py --workload cfg1 --no-cpu-baseline > $OUT/bench_cfg1.log 2>&1

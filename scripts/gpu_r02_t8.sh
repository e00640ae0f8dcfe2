#!/bin/bash
OUT=gpurun_out/r02_t8
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for w in 1 2 4 8; do
  timeout 900 python bench.py --workload sweep --workers $w --no-cpu-baseline > $OUT/bench_sweep_w$w.log 2>&1
  cp -f gpurun_out/sweep_w1.log $OUT/sweep_workers$w.log
done
timeout 900 python scripts/sweep_kernels.py 1024 > $OUT/sweep_kernels.txt 2>&1
timeout 600 python bench.py > $OUT/bench_resnet18.log 2>&1

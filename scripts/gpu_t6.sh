#!/bin/bash
OUT=gpurun_out/${1:-t6}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python scripts/sweep_fail.py 8 170 518 732 828 > $OUT/sweep_fail.txt 2>&1
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep.log 2>&1
cp gpurun_out/sweep_rank0.log $OUT/ 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_resnet18.log 2>&1

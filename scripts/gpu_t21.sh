#!/bin/bash
OUT=gpurun_out/${1:-t21}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep.log 2>&1
cp gpurun_out/sweep_rank0.log $OUT/ 2>/dev/null

#!/bin/bash
OUT=gpurun_out/r02_t6
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep.log 2>&1
cp -f gpurun_out/sweep_w1.log $OUT/sweep_conc.log
timeout 900 python bench.py --workload sweep --workers 1 --steps 1 --no-cpu-baseline > $OUT/bench_sweep_serial.log 2>&1
cp -f gpurun_out/sweep_w1.log $OUT/sweep_serial.log 2>/dev/null
timeout 900 python scripts/sweep_kernels.py 1024 > $OUT/sweep_kernels.txt 2>&1

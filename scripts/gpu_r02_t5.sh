#!/bin/bash
# Gathered GEMM on tcgen05: parity + sweep timing.
OUT=gpurun_out/r02_t5
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gathered" > $OUT/pytest_gg.log 2>&1; echo "rc=$?" >> $OUT/pytest_gg.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reward.py tests/test_gpu_reference_objects.py -m gpu -q > $OUT/pytest_parity.log 2>&1; echo "rc=$?" >> $OUT/pytest_parity.log
timeout 900 python bench.py --workload sweep --workers 1 --steps 1 --no-cpu-baseline > $OUT/bench_sweep_serial.log 2>&1
cp -f gpurun_out/sweep_w1.log $OUT/sweep_serial.log 2>/dev/null
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep.log 2>&1
timeout 900 python scripts/sweep_kernels.py 1024 > $OUT/sweep_kernels.txt 2>&1

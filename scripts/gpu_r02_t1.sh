#!/bin/bash
# New parity tests at bench shapes + heavy candidates; bench lines with the honest roofline.
OUT=gpurun_out/r02_t1
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_bench_shapes.py tests/test_gpu_parity.py -m gpu -q -x -k "bench_shape or resnet or qkv or pointwise or fallback or full_size or heavy or staged_fp32" > $OUT/pytest_new.log 2>&1; echo "rc=$?" >> $OUT/pytest_new.log
timeout 600 python bench.py > $OUT/bench_resnet18.log 2>&1
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep.log 2>&1
cp -f gpurun_out/sweep_w1.log $OUT/ 2>/dev/null
timeout 900 python bench.py --workload sweep --workers 1 --steps 1 --no-cpu-baseline > $OUT/bench_sweep_serial.log 2>&1
cp -f gpurun_out/sweep_w1.log $OUT/sweep_serial.log 2>/dev/null

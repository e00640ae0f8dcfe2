#!/bin/bash
OUT=gpurun_out/${1:-t7}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_resnet18.log 2>&1
SYNO_NO_PDL=1 timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_resnet18_nopdl.log 2>&1
timeout 600 python bench.py --workload cfg1 --no-cpu-baseline > $OUT/bench_cfg1.log 2>&1
timeout 600 python bench.py --workload qkv --no-cpu-baseline > $OUT/bench_qkv.log 2>&1
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep.log 2>&1

#!/bin/bash
OUT=gpurun_out/${1:-t12}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
bash scripts/gpu_attrib.sh ${1:-t12}
timeout 600 python bench.py --workload resnet34 --steps 5 --no-cpu-baseline > $OUT/bench_resnet34.log 2>&1
timeout 600 python bench.py --workload qkv --no-cpu-baseline > $OUT/bench_qkv.log 2>&1

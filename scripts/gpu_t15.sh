#!/bin/bash
OUT=gpurun_out/${1:-t15}
mkdir -p $OUT
timeout 600 python bench.py > $OUT/bench_resnet18.log 2>&1
timeout 600 python bench.py --workload resnet34 --steps 5 --no-cpu-baseline > $OUT/bench_resnet34.log 2>&1
timeout 600 python bench.py --workload qkv --no-cpu-baseline > $OUT/bench_qkv.log 2>&1
timeout 600 python bench.py --workload cfg1 --no-cpu-baseline > $OUT/bench_cfg1.log 2>&1

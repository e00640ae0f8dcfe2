#!/bin/bash
# Bench all workloads once (one gpurun call).  usage: bash scripts/gpu_bench.sh <tag>
TAG=${1:-r01b}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python bench.py > $OUT/bench_resnet18.log 2>&1; echo "rc=$?" >> $OUT/bench_resnet18.log
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep.log 2>&1; echo "rc=$?" >> $OUT/bench_sweep.log
timeout 600 python bench.py --workload qkv_train --steps 5 > $OUT/bench_qkv_train.log 2>&1; echo "rc=$?" >> $OUT/bench_qkv_train.log
timeout 600 python bench.py --workload cfg1 --no-cpu-baseline > $OUT/bench_cfg1.log 2>&1; echo "rc=$?" >> $OUT/bench_cfg1.log
timeout 600 python bench.py --workload resnet34 --no-cpu-baseline --steps 5 > $OUT/bench_resnet34.log 2>&1; echo "rc=$?" >> $OUT/bench_resnet34.log
timeout 600 python bench.py --workload qkv --no-cpu-baseline > $OUT/bench_qkv.log 2>&1; echo "rc=$?" >> $OUT/bench_qkv.log
ls -la $OUT

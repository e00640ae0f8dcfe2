#!/bin/bash
# Round-end bench lines only (no ncu): GPU tests, smoke, every workload's JSON line.
OUT=gpurun_out/${1:-benches}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_resnet18.log 2>&1
timeout 600 python bench.py --impl reference --steps 1 > $OUT/bench_reference.log 2>&1
timeout 600 python bench.py --workload resnet34 --steps 5 --no-cpu-baseline > $OUT/bench_resnet34.log 2>&1
timeout 600 python bench.py --workload qkv --no-cpu-baseline > $OUT/bench_qkv.log 2>&1
timeout 600 python bench.py --workload cfg1 > $OUT/bench_cfg1.log 2>&1
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep.log 2>&1
timeout 600 python bench.py --workload qkv_train --steps 20 > $OUT/bench_qkv_train.log 2>&1
tail -2 $OUT/pytest_gpu.log

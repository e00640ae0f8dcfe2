#!/bin/bash
# Round-2 state capture: smoke, GPU tests, every bench workload, reference arm, ncu launch list.
OUT=gpurun_out/${1:-r02_state}
mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
for w in resnet18 qkv resnet34 cfg1; do
  timeout 600 python bench.py --workload $w > $OUT/bench_$w.log 2>&1
done
timeout 900 python bench.py --workload sweep > $OUT/bench_sweep.log 2>&1
cp -f gpurun_out/sweep_rank0.log $OUT/ 2>/dev/null
timeout 600 python bench.py --workload qkv_train --no-cpu-baseline > $OUT/bench_qkv_train.log 2>&1
timeout 600 python bench.py --impl reference > $OUT/bench_reference.log 2>&1
#timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_resnet18.csv \
#  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > $OUT/ncu_bench.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log

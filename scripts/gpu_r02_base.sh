#!/bin/bash
# Round-2 starting point: GPU tests, default bench, sweep log (per-candidate failures).
OUT=gpurun_out/r02_base
mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_resnet18.log 2>&1
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep.log 2>&1
cp -f gpurun_out/sweep_rank0.log $OUT/ 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log

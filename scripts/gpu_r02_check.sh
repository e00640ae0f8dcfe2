#!/bin/bash
# GPU tests + default bench + sweep bench of the current tree.
OUT=gpurun_out/${1:-r02_check}
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_resnet18.log 2>&1
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep.log 2>&1
cp -f gpurun_out/sweep_w1.log $OUT/ 2>/dev/null

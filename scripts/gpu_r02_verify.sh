#!/bin/bash
# Last check of HEAD: smoke, GPU suite, the default bench line, proxy training.
OUT=gpurun_out/${1:-r02_verify}
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_default.log 2>&1
timeout 600 python bench.py --workload qkv_train --no-cpu-baseline > $OUT/bench_qkv_train.log 2>&1

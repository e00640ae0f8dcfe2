#!/bin/bash
# Lane-contiguous permuted copies (default) vs none (SYNO_NO_PERM=1): parity, heavy candidates, sweep.
OUT=gpurun_out/r02_perm
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_shapes.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
IDS="828 170 961 796 688 404 732 247 12 331 284 125"
timeout 600 python scripts/sweep_prof_one.py $IDS > $OUT/perm.txt 2>&1
SYNO_NO_PERM=1 timeout 600 python scripts/sweep_prof_one.py $IDS > $OUT/noperm.txt 2>&1
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep_perm.log 2>&1
cp -f gpurun_out/sweep_w1.log $OUT/sweep_perm.log
SYNO_NO_PERM=1 timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep_noperm.log 2>&1

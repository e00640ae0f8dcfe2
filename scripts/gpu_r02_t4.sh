#!/bin/bash
# Tiled scatter: parity + sweep timing; pack-kernel ncu capture of the ResNet-18 step.
OUT=gpurun_out/r02_t4
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reward.py tests/test_gpu_reference_objects.py -m gpu -q -x > $OUT/pytest_parity.log 2>&1; echo "rc=$?" >> $OUT/pytest_parity.log
timeout 900 python bench.py --workload sweep --workers 1 --steps 1 --no-cpu-baseline > $OUT/bench_sweep_serial.log 2>&1
cp -f gpurun_out/sweep_w1.log $OUT/sweep_serial.log 2>/dev/null
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep.log 2>&1
timeout 900 python scripts/sweep_kernels.py 1024 > $OUT/sweep_kernels.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"prep_kernel|pack_rows" -c 27 -o /tmp/pack_full \
    python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline > $OUT/ncu_pack.log 2>&1
ncu -i /tmp/pack_full.ncu-rep --page raw --csv > $OUT/pack_raw.csv 2>/dev/null

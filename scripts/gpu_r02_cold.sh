#!/bin/bash
OUT=gpurun_out/r02_cold
mkdir -p $OUT
IDS="124 179 21 404 828 688 170 961 796 732 247 12 319 73 15 381"
timeout 600 python scripts/sweep_cold.py $IDS > $OUT/pool.txt 2>&1
SYNO_TC_SYNC_ALLOC=1 timeout 600 python scripts/sweep_cold.py $IDS > $OUT/sync.txt 2>&1
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep_pool.log 2>&1
cp gpurun_out/sweep_w1.log $OUT/sweep_pool.log

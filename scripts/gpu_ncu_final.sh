#!/bin/bash
# Round-end ncu evidence of the default bench: launch list + one --set full capture of the tc_gemm launches.
OUT=gpurun_out/${1:-ncu_final}
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline > $OUT/ncu_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:tc_gemm -c 60 -o /tmp/tc_full \
    python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline > $OUT/ncu_full.log 2>&1
ncu -i /tmp/tc_full.ncu-rep --page raw --csv > $OUT/tc_full_raw.csv 2>/dev/null
bash scripts/gpu_attrib.sh $(basename $OUT)
ls $OUT

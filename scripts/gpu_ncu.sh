#!/bin/bash
# ncu evidence for the default bench: launch list (all kernels, serialised,
# cold-cache) and one --set full capture of the tc_gemm launches of a step.
OUT=gpurun_out/${1:-ncu}
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline > $OUT/ncu_launch_bench.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 60 -o $OUT/tc_full \
    python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline > $OUT/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"pack_rows|fold_tile|chain_n|cast_f32" -c 12 -o $OUT/aux_full \
    python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline > $OUT/ncu_aux.log 2>&1
ls -la $OUT

#!/bin/bash
# ncu evidence for the default bench, post-processed on the box (reports stay small).
OUT=gpurun_out/${1:-ncu}
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline > $OUT/ncu_launch_bench.log 2>&1
# one full capture of the first step's 60 tc_gemm launches (no source page: keeps the report small)
timeout 1500 ncu --set full --clock-control none -k regex:tc_gemm -c 60 -o /tmp/tc_full \
    python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline > $OUT/ncu_full.log 2>&1
ncu -i /tmp/tc_full.ncu-rep --page raw --csv > $OUT/tc_full_raw.csv 2>/dev/null
ncu -i /tmp/tc_full.ncu-rep --page details --csv > $OUT/tc_full_details.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:"pack_rows|fold_tile|chain_n|cast_f32|zero_fill" -c 10 -o /tmp/aux_full \
    python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline > $OUT/ncu_aux.log 2>&1
ncu -i /tmp/aux_full.ncu-rep --page details --csv > $OUT/aux_full_details.csv 2>/dev/null
ncu -i /tmp/aux_full.ncu-rep --page raw --csv > $OUT/aux_full_raw.csv 2>/dev/null
# a small source-annotated capture of one forward GEMM of layer1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 -o $OUT/tc_one \
    python scripts/gemm_probe.py conv3x3 64 64 32 128 1 > $OUT/ncu_one.log 2>&1
du -sh $OUT; ls -la $OUT

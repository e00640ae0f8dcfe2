#!/bin/bash
OUT=gpurun_out/${1:-t10}
mkdir -p $OUT
timeout 120 python scripts/gemm_probe.py conv3x3 512 512 4 128 10 >> $OUT/probe.txt 2>&1
SYNO_TC_ZERO_FILL=1 timeout 120 python scripts/gemm_probe.py conv3x3 512 512 4 128 10 >> $OUT/probe.txt 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"chain_nc|fold_tile|zero_fill" -c 6 -o /tmp/ch python scripts/gemm_probe.py conv3x3 512 512 4 128 1 > $OUT/ncu.log 2>&1
ncu -i /tmp/ch.ncu-rep --page details --csv > $OUT/ch_details.csv 2>/dev/null

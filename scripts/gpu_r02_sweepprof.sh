#!/bin/bash
OUT=gpurun_out/r02_sweepprof
mkdir -p $OUT
IDS="124 179 21 404 828 688 170 961 796 732 247 12"
timeout 600 python scripts/sweep_prof_one.py $IDS > $OUT/gg.txt 2>&1
SYNO_NO_GATHER_GEMM=1 timeout 600 python scripts/sweep_prof_one.py $IDS > $OUT/nogg.txt 2>&1

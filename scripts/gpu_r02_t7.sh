#!/bin/bash
OUT=gpurun_out/r02_t7
mkdir -p $OUT
timeout 600 python scripts/sweep_prof.py 1024 > $OUT/sweep_prof_serial.txt 2>&1
timeout 600 python scripts/sweep_prof_conc.py 1 > $OUT/sweep_prof_w1.txt 2>&1
timeout 600 python scripts/sweep_prof_conc.py 8 > $OUT/sweep_prof_w8.txt 2>&1

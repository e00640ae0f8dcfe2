#!/bin/bash
# One source-annotated ncu capture of a GEMM launch of one layer (for stall attribution per SASS line).
OUT=gpurun_out/${1:-ncu_src}
shift
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 -o $OUT/rep \
    python scripts/gemm_probe.py "$@" > $OUT/ncu.log 2>&1
ncu -i $OUT/rep.ncu-rep --page source --csv --print-source sass > $OUT/src.csv 2>/dev/null
ncu -i $OUT/rep.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ls -la $OUT

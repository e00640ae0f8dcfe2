#!/bin/bash
# ncu --set full (source-annotated) of the first launch of kernel regex $2 in `gemm_probe.py ${@:3}`.
OUT=gpurun_out/$1
KRE=$2
shift 2
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KRE -c 1 -o $OUT/rep \
    python scripts/gemm_probe.py "$@" > $OUT/ncu.log 2>&1
ncu -i $OUT/rep.ncu-rep --page source --csv --print-source sass > $OUT/src.csv 2>/dev/null
ncu -i $OUT/rep.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ls -la $OUT

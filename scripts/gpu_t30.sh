#!/bin/bash
# ncu source-level warp-stall sampling of the forward GEMM (64->64 @32, N=128)
OUT=gpurun_out/${1:-t30}
mkdir -p $OUT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 3 -c 1 -o /tmp/g64 \
  python scripts/gemm_probe.py conv3x3 64 64 32 128 1 > $OUT/ncu.log 2>&1
ncu -i /tmp/g64.ncu-rep --page source --csv --print-source sass > $OUT/src_sass.csv 2>/dev/null
ncu -i /tmp/g64.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ncu -i /tmp/g64.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ls -la $OUT

#!/bin/bash
# Stem / l1 / l4 layer investigation: tiling log, per-class times, one source-annotated
# ncu capture of the stem forward GEMM and of the l1 forward GEMM.
OUT=gpurun_out/r02_stem
mkdir -p $OUT
for L in "conv3x3 3 64 32 128" "conv3x3 64 64 32 128" "sep_shared 64 64 32 128" "conv3x3 512 512 4 128"; do
  SYNO_TC_LOG=1 timeout 300 python scripts/gemm_probe.py $L > "$OUT/probe_${L// /_}.log" 2>&1
done
for L in "conv3x3 3 64 32 128" "conv3x3 64 64 32 128"; do
  n=${L// /_}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -o $OUT/rep_$n \
    python scripts/gemm_probe.py $L 2 > $OUT/ncu_$n.log 2>&1
  ncu -i $OUT/rep_$n.ncu-rep --page source --csv --print-source sass > $OUT/src_$n.csv 2>/dev/null
  ncu -i $OUT/rep_$n.ncu-rep --page details --csv > $OUT/details_$n.csv 2>/dev/null
  rm -f $OUT/rep_$n.ncu-rep
done

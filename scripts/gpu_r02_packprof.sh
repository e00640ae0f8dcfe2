#!/bin/bash
# ncu --set full of the operand packs of an l1 (64ch @32, N=128) and an l3 (256ch @8) layer.
OUT=gpurun_out/r02_packprof
mkdir -p $OUT
for L in "conv3x3 64 64 32 128" "conv3x3 256 256 8 128"; do
  n=${L// /_}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prep_kernel|pack_rows" -s 3 -c 3 -o $OUT/rep_$n \
    python scripts/gemm_probe.py $L 2 > $OUT/ncu_$n.log 2>&1
  ncu -i $OUT/rep_$n.ncu-rep --page details --csv > $OUT/details_$n.csv 2>/dev/null
  ncu -i $OUT/rep_$n.ncu-rep --page source --csv --print-source sass > $OUT/src_$n.csv 2>/dev/null
  rm -f $OUT/rep_$n.ncu-rep
done

#!/bin/bash
# ncu --set full of the chain-rule kernels of sep_shared / conv3x3 layers (ResNet-18 shapes).
OUT=gpurun_out/r02_chain
mkdir -p $OUT
for L in "sep_shared 64 64 32 128" "sep_shared 512 512 4 128" "conv3x3 512 512 4 128"; do
  n=${L// /_}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain -s 2 -c 1 -o $OUT/rep_$n \
    python scripts/gemm_probe.py $L 2 > $OUT/ncu_$n.log 2>&1
  ncu -i $OUT/rep_$n.ncu-rep --page source --csv --print-source sass > $OUT/src_$n.csv 2>/dev/null
  ncu -i $OUT/rep_$n.ncu-rep --page details --csv > $OUT/details_$n.csv 2>/dev/null
  rm -f $OUT/rep_$n.ncu-rep
done

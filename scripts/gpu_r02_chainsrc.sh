#!/bin/bash
# Dense-sampled source profile of the small sep_shared chain (chain_v4) and chain_win (64 x 64 layers).
OUT=gpurun_out/r02_chainsrc
mkdir -p $OUT
for L in "sep_shared 64 64 32 128" "conv3x3 64 64 32 128"; do
  n=${L// /_}
  timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:chain -s 2 -c 1 \
    -o $OUT/rep_$n python scripts/gemm_probe.py $L 2 > $OUT/ncu_$n.log 2>&1
  ncu -i $OUT/rep_$n.ncu-rep --page source --csv --print-source sass > $OUT/src_$n.csv 2>/dev/null
  ncu -i $OUT/rep_$n.ncu-rep --page details --csv > $OUT/details_$n.csv 2>/dev/null
  ncu -i $OUT/rep_$n.ncu-rep --page raw --csv > $OUT/raw_$n.csv 2>/dev/null
  rm -f $OUT/rep_$n.ncu-rep
done

#!/bin/bash
# GEMM bottleneck switches on one layer: SYNO_TC_DEBUG 1 no stores, 2 no MMAs, 4/8 no A/B loads, 256 no TMEM reads or stores.
OUT=gpurun_out/${1:-dbg}
shift
mkdir -p $OUT
for d in ${DBGS:-0 1 256 2 12 14 270}; do
  echo "### dbg=$d" >> $OUT/dbg.txt
  SYNO_TC_PAIR=0 SYNO_TC_DEBUG=$d timeout 120 python scripts/gemm_probe.py "$@" 2>&1 | grep tc_gemm >> $OUT/dbg.txt
done
cat $OUT/dbg.txt

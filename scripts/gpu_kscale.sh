#!/bin/bash
# GEMM skeleton cost vs k-steps per tile: pointwise 1x1 operators (M = 16384 pixels, N = 2304) with C_in 64..768,
# DBG build, switches 0 (full) and 270 (no loads, MMAs, epilogue work).
OUT=gpurun_out/${1:-kscale}
mkdir -p $OUT
touch paper_2410_23745_b200/csrc/tc.cu && make DBG=1 -j8 > $OUT/build.log 2>&1
for cin in 64 256 768; do
  for d in 0 270; do
    echo "### cin=$cin dbg=$d $(SYNO_TC_PAIR=0 SYNO_TC_DEBUG=$d timeout 120 python scripts/gemm_probe.py pointwise $cin 2304 128 1 5 2>&1 | grep -E '^  tc_gemm_fwd' | tr '\n' ' ')" >> $OUT/k.txt
  done
done
touch paper_2410_23745_b200/csrc/tc.cu && make -j8 > /dev/null 2>&1
cat $OUT/k.txt

#!/bin/bash
# Event trace (TRACE=1 DBG=1 build) of the conv3x3 64->64 @32 N=128 forward GEMM under switch sets $DBGS.
OUT=gpurun_out/${1:-trace_conv}
mkdir -p $OUT
touch paper_2410_23745_b200/csrc/tc.cu && make TRACE=1 DBG=1 -j8 > $OUT/build.log 2>&1
for dbg in ${DBGS:-270}; do
  SYNO_TC_DEBUG=$dbg SYNO_TC_TRACE=$OUT/trace_$dbg.txt timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 1 > /dev/null 2>&1
done
touch paper_2410_23745_b200/csrc/tc.cu && make DBG=1 -j8 > /dev/null 2>&1
for dbg in ${DBGS:-270}; do
  echo "### dbg=$dbg $(SYNO_TC_DEBUG=$dbg timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 5 2>&1 | grep tc_gemm_fwd)" >> $OUT/t.txt
done
touch paper_2410_23745_b200/csrc/tc.cu && make -j8 > /dev/null 2>&1
cat $OUT/t.txt

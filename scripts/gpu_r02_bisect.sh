#!/bin/bash
# Window-issue period of the conv3x3 64->64 @32 forward GEMM under bottleneck switches (TRACE+DBG build).
OUT=gpurun_out/r02_bisect
mkdir -p $OUT
touch paper_2410_23745_b200/csrc/tc.cu && make TRACE=1 DBG=1 -j8 > $OUT/build.log 2>&1
for dbg in 0 261 1 4 256 257 64 320; do
  SYNO_TC_SMALL=0 SYNO_TC_G=1 SYNO_TC_DEBUG=$dbg SYNO_TC_TRACE=$OUT/trace_$dbg.txt timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 1 > /dev/null 2>&1
done
touch paper_2410_23745_b200/csrc/tc.cu && make -j8 > /dev/null 2>&1

#!/bin/bash
# Event trace (TRACE=1 build) of the QKV forward GEMM, with and without the bottleneck switches.
OUT=gpurun_out/${1:-trace_qkv}
mkdir -p $OUT
touch paper_2410_23745_b200/csrc/tc.cu && make TRACE=1 ${XMAKE} -j8 > $OUT/build.log 2>&1
for dbg in ${DBGS:-0}; do
  SYNO_TC_PAIR=${PAIR:-0} SYNO_TC_DEBUG=$dbg SYNO_TC_TRACE=$OUT/trace_$dbg.txt timeout 120 python scripts/gemm_probe.py qkv 768 2304 1024 16 1 > /dev/null 2>&1
  python scripts/trace_view.py $OUT/trace_$dbg.txt 0 > $OUT/view_$dbg.txt 2>&1
  python scripts/trace_raw.py $OUT/trace_$dbg.txt 0 "" 2 > $OUT/raw_$dbg.txt 2>&1
done
touch paper_2410_23745_b200/csrc/tc.cu && make -j8 > /dev/null 2>&1
head -30 $OUT/view_0.txt $OUT/view_270.txt

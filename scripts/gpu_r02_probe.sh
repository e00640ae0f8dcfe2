#!/bin/bash
# Round-2 GEMM investigation: per-layer kernel classes (current build) and an
# event trace of the conv3x3 64->64 @32 N=128 forward GEMM.
OUT=gpurun_out/r02_probe
mkdir -p $OUT
for args in "stem:conv3x3 3 64 32 128" "l1:conv3x3 64 64 32 128" "l1s:sep_shared 64 64 32 128" "l2:conv3x3 128 128 16 128" \
            "l3:conv3x3 256 256 8 128" "l4:conv3x3 512 512 4 128" "s2:conv3x3_s2 64 128 16 128" "sc:shortcut_s2 64 128 16 128"; do
  name=${args%%:*}; a=${args#*:}
  timeout 120 python scripts/gemm_probe.py $a 10 > $OUT/probe_$name.txt 2>&1
done
SYNO_TC_LOG=1 timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 1 > $OUT/log_l1.txt 2>&1
SYNO_TC_LOG=1 timeout 120 python scripts/gemm_probe.py conv3x3 3 64 32 128 1 > $OUT/log_stem.txt 2>&1
SYNO_TC_LOG=1 timeout 120 python scripts/gemm_probe.py shortcut_s2 64 128 16 128 1 > $OUT/log_sc.txt 2>&1
touch paper_2410_23745_b200/csrc/tc.cu && make TRACE=1 DBG=1 -j8 > $OUT/build.log 2>&1
for dbg in 0 270; do
  SYNO_TC_DEBUG=$dbg SYNO_TC_TRACE=$OUT/trace_$dbg.txt timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 1 > /dev/null 2>&1
done
touch paper_2410_23745_b200/csrc/tc.cu && make -j8 > /dev/null 2>&1

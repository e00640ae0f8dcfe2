#!/bin/bash
# A/B of GEMM configuration switches on the ResNet-18 layer shapes (per-kernel, serialised).
OUT=gpurun_out/r02_ab
mkdir -p $OUT
for cfg in "base:" "small0:SYNO_TC_SMALL=0" "small0g1:SYNO_TC_SMALL=0 SYNO_TC_G=1" "small0g2:SYNO_TC_SMALL=0 SYNO_TC_G=2" \
           "nobres:SYNO_TC_NO_BRES=1" "nobres_s0g1:SYNO_TC_NO_BRES=1 SYNO_TC_SMALL=0 SYNO_TC_G=1"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  for args in "conv3x3 64 64 32 128" "conv3x3 128 128 16 128" "conv3x3 256 256 8 128" "conv3x3 3 64 32 128" "shortcut_s2 64 128 16 128"; do
    echo "## $name $args" >> $OUT/ab.txt
    env $envs timeout 120 python scripts/gemm_probe.py $args 10 2>&1 | grep tc_gemm >> $OUT/ab.txt
  done
done
touch paper_2410_23745_b200/csrc/tc.cu && make TRACE=1 DBG=1 -j8 > $OUT/build.log 2>&1
SYNO_TC_SMALL=0 SYNO_TC_G=1 SYNO_TC_TRACE=$OUT/trace_s0g1.txt timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 1 > /dev/null 2>&1
SYNO_TC_TRACE=$OUT/trace_sc.txt timeout 120 python scripts/gemm_probe.py shortcut_s2 64 128 16 128 1 > /dev/null 2>&1
SYNO_TC_TRACE=$OUT/trace_stem.txt timeout 120 python scripts/gemm_probe.py conv3x3 3 64 32 128 1 > /dev/null 2>&1
touch paper_2410_23745_b200/csrc/tc.cu && make -j8 > /dev/null 2>&1

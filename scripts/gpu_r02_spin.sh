#!/bin/bash
OUT=gpurun_out/r02_spin
mkdir -p $OUT
timeout 120 ./scripts/mwb > $OUT/mwb.txt 2>&1
for args in "conv3x3 64 64 32 128" "conv3x3 128 128 16 128" "conv3x3 256 256 8 128"; do
  echo "## base $args" >> $OUT/ab.txt; timeout 120 python scripts/gemm_probe.py $args 10 2>&1 | grep tc_gemm >> $OUT/ab.txt
done
touch paper_2410_23745_b200/csrc/tc.cu && make SUSPEND=1 -j8 > $OUT/build.log 2>&1
for args in "conv3x3 64 64 32 128" "conv3x3 128 128 16 128" "conv3x3 256 256 8 128"; do
  echo "## suspend $args" >> $OUT/ab.txt; timeout 120 python scripts/gemm_probe.py $args 10 2>&1 | grep tc_gemm >> $OUT/ab.txt
done
timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_suspend.log 2>&1
touch paper_2410_23745_b200/csrc/tc.cu && make -j8 > /dev/null 2>&1

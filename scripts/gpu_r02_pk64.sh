#!/bin/bash
# Pack block size A/B: PK_PIX=128 (libsyno.so) vs 64 (libsyno_pk64.so, SYNO_LIB_PATH); tests on the variant.
OUT=gpurun_out/r02_pk64
mkdir -p $OUT
V=$PWD/paper_2410_23745_b200/libsyno_pk64.so
for L in "conv3x3 64 64 32 128" "conv3x3 256 256 8 128" "conv3x3 128 128 56 256"; do
  n=${L// /_}
  timeout 300 python scripts/gemm_probe.py $L > $OUT/probe_$n.log 2>&1
  SYNO_LIB_PATH=$V timeout 300 python scripts/gemm_probe.py $L > $OUT/probe_pk64_$n.log 2>&1
done
for i in 1 2; do
  timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_r18_$i.log 2>&1
  SYNO_LIB_PATH=$V timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_r18_pk64_$i.log 2>&1
done
timeout 600 python bench.py --workload resnet34 --no-cpu-baseline > $OUT/bench_r34.log 2>&1
SYNO_LIB_PATH=$V timeout 600 python bench.py --workload resnet34 --no-cpu-baseline > $OUT/bench_r34_pk64.log 2>&1
SYNO_LIB_PATH=$V timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_pk64.log 2>&1; echo "rc=$?" >> $OUT/pytest_pk64.log

#!/bin/bash
# Stem channel padding A/B (SYNO_TC_CP_MIN): per-class times of the 3-channel stem, its bench-shape
# parity test under each setting, and the ResNet-18 step.
OUT=gpurun_out/r02_cpmin
mkdir -p $OUT
for cp in 0 16 32 64; do
  SYNO_TC_CP_MIN=$cp timeout 300 python scripts/gemm_probe.py conv3x3 3 64 32 128 > $OUT/probe_cp$cp.log 2>&1
  SYNO_TC_CP_MIN=$cp timeout 600 python -m pytest tests/test_gpu_bench_shapes.py -q -x -k "stem" > $OUT/pytest_cp$cp.log 2>&1
  echo "rc=$?" >> $OUT/pytest_cp$cp.log
done
for i in 1 2; do
  for cp in 0 64; do
    SYNO_TC_CP_MIN=$cp timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_cp${cp}_$i.log 2>&1
  done
done

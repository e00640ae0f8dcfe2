#!/bin/bash
OUT=gpurun_out/${1:-t4}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for cfg in "conv3x3 64 64 32 128" "sep_shared 64 64 32 128" "conv3x3 512 512 4 128" "qkv 0 0 0 16"; do
  timeout 120 python scripts/gemm_probe.py $cfg 10 >> $OUT/probe.txt 2>&1
done
timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 8 10 float32 >> $OUT/probe.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_resnet18.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:pack_rows -c 2 -o $OUT/pack python scripts/gemm_probe.py conv3x3 64 64 32 128 1 > $OUT/ncu_pack.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"fold_tile|chain_n" -c 4 -o $OUT/wt python scripts/gemm_probe.py conv3x3 512 512 4 128 1 > $OUT/ncu_wt.log 2>&1

#!/bin/bash
# QKV GEMM investigation: MMA issue-rate microbenchmark, per-launch probe, one ncu capture of each GEMM role.
OUT=gpurun_out/${1:-qkv}
mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2410_23745_b200/csrc scripts/mma_bench.cu -o /tmp/mma_bench -lcuda \
  && timeout 120 /tmp/mma_bench > $OUT/mma_bench.txt 2>&1
timeout 300 python scripts/gemm_probe.py qkv 768 2304 1024 16 10 > $OUT/probe_qkv.txt 2>&1
SYNO_TC_LOG=1 timeout 300 python scripts/gemm_probe.py qkv 768 2304 1024 16 1 > $OUT/probe_qkv_log.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 3 -o $OUT/tc_qkv \
    python scripts/gemm_probe.py qkv 768 2304 1024 16 1 > $OUT/ncu_qkv.log 2>&1
ncu -i $OUT/tc_qkv.ncu-rep --page raw --csv > $OUT/tc_qkv_raw.csv 2>/dev/null
ncu -i $OUT/tc_qkv.ncu-rep --page details --csv > $OUT/tc_qkv_details.csv 2>/dev/null
ls -la $OUT

#!/bin/bash
# CTA-pair GEMM bring-up: tc parity tests, probes with the configuration log, QKV / ResNet-34 benches.
OUT=gpurun_out/${1:-pair}
mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q > $OUT/pytest_tc.log 2>&1; echo "rc=$?" >> $OUT/pytest_tc.log
SYNO_TC_LOG=1 timeout 120 python scripts/gemm_probe.py qkv 768 2304 1024 16 1 2>&1 | grep -E "gemm|TF" > $OUT/probe_qkv_log.txt
timeout 120 python scripts/gemm_probe.py qkv 768 2304 1024 16 10 > $OUT/probe_qkv.txt 2>&1
SYNO_TC_PAIR=0 timeout 120 python scripts/gemm_probe.py qkv 768 2304 1024 16 10 > $OUT/probe_qkv_nopair.txt 2>&1
timeout 120 python scripts/gemm_probe.py conv3x3 256 256 14 256 10 > $OUT/probe_c256.txt 2>&1
SYNO_TC_PAIR=0 timeout 120 python scripts/gemm_probe.py conv3x3 256 256 14 256 10 > $OUT/probe_c256_nopair.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --workload qkv --no-cpu-baseline > $OUT/bench_qkv.log 2>&1
timeout 600 python bench.py --workload resnet34 --steps 5 --no-cpu-baseline > $OUT/bench_resnet34.log 2>&1
tail -3 $OUT/pytest_tc.log

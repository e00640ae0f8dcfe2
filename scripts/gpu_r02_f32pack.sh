#!/bin/bash
# fp32 pack read phase with all loads in flight: cfg1 bench, fp32 per-class times, full GPU suite.
OUT=gpurun_out/r02_f32pack
mkdir -p $OUT
timeout 300 python scripts/gemm_probe.py conv3x3 64 64 32 8 10 float32 > $OUT/probe_cfg1.log 2>&1
for i in 1 2; do timeout 600 python bench.py --workload cfg1 > $OUT/bench_cfg1_$i.log 2>&1; done
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_default.log 2>&1

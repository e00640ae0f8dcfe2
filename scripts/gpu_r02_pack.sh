#!/bin/bash
OUT=gpurun_out/r02_pack
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_bench_shapes.py tests/test_gpu_parity.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 10 > $OUT/probe_l1.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > $OUT/bench18.log 2>&1
timeout 300 python bench.py --workload resnet34 --no-cpu-baseline > $OUT/bench34.log 2>&1
timeout 120 python scripts/link_bw.py 512 > $OUT/link.txt 2>&1

#!/bin/bash
OUT=gpurun_out/${1:-t14}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
bash scripts/gpu_ks.sh ${1:-t14}
bash scripts/gpu_attrib.sh ${1:-t14}

#!/bin/bash
# The driver's default bench run (with other_configs), twice.
OUT=gpurun_out/${1:-r02_default}
mkdir -p $OUT
for i in 1 2; do timeout 900 python bench.py > $OUT/bench_default_$i.log 2>&1; done

#!/bin/bash
# Round-end evidence: all bench workloads + attribution + ncu launch list.
OUT=gpurun_out/${1:-final}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_resnet18.log 2>&1
timeout 600 python bench.py --impl reference --steps 1 > $OUT/bench_reference.log 2>&1
timeout 600 python bench.py --workload resnet34 --steps 5 --no-cpu-baseline > $OUT/bench_resnet34.log 2>&1
timeout 600 python bench.py --workload qkv --no-cpu-baseline > $OUT/bench_qkv.log 2>&1
timeout 600 python bench.py --workload cfg1 > $OUT/bench_cfg1.log 2>&1
timeout 900 python bench.py --workload sweep --no-cpu-baseline > $OUT/bench_sweep.log 2>&1
timeout 600 python bench.py --workload qkv_train --steps 5 > $OUT/bench_qkv_train.log 2>&1
bash scripts/gpu_attrib.sh ${1:-final}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline > $OUT/ncu_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:tc_gemm -c 60 -o /tmp/tc_full \
    python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline > $OUT/ncu_full.log 2>&1
ncu -i /tmp/tc_full.ncu-rep --page raw --csv > $OUT/tc_full_raw.csv 2>/dev/null
ncu -i /tmp/tc_full.ncu-rep --page details --csv > $OUT/tc_full_details.csv 2>/dev/null
du -sh $OUT

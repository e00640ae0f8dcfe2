#!/bin/bash
# End-of-round capture: smoke, the default bench line (with other_configs), every workload's own line,
# the reference arm, the ResNet-18 ncu launch list and --set full GEMM capture, the GPU suite.
OUT=gpurun_out/${1:-r02_final}
mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.log 2>&1
for w in resnet34 qkv cfg1; do
  timeout 600 python bench.py --workload $w > $OUT/bench_$w.log 2>&1
done
timeout 900 python bench.py --workload sweep > $OUT/bench_sweep.log 2>&1
cp -f gpurun_out/sweep_w1.log $OUT/ 2>/dev/null
timeout 600 python bench.py --workload qkv_train --no-cpu-baseline > $OUT/bench_qkv_train.log 2>&1
timeout 600 python bench.py --impl reference > $OUT/bench_reference.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:tc_gemm -c 60 -o $OUT/r18 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-others > $OUT/ncu_r18.log 2>&1
ncu -i $OUT/r18.ncu-rep --page raw --csv > $OUT/r18_raw.csv 2>/dev/null
rm -f $OUT/r18.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches_r18.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-others > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log

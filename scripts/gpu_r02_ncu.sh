#!/bin/bash
# ncu --set full of the dominant kernel of each layer workload (one step, eager launches)
# and the launch list of each; summaries -> profiles/ via scripts/ncu_summary.py.
OUT=gpurun_out/r02_ncu
mkdir -p $OUT
for w in resnet18:60 resnet34:105 qkv:3 cfg1:1; do
  name=${w%%:*}; n=${w#*:}
  timeout 1200 ncu --set full --clock-control none -k regex:tc_gemm -c $n -o $OUT/$name \
    python bench.py --workload $name --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $OUT/ncu_$name.log 2>&1
  ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches_$name.csv \
    python bench.py --workload $name --steps 1 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
done
rm -f $OUT/*.ncu-rep

#!/bin/bash
OUT=gpurun_out/${1:-chp}
mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum --cache-control none --clock-control none -k regex:"chain|fold|pack" --csv --log-file $OUT/aux.csv \
    python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline > $OUT/log.txt 2>&1

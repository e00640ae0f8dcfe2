#!/bin/bash
OUT=gpurun_out/r02_t9
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stage_tile" -c 12 -o /tmp/tile_full \
    python scripts/sweep_one.py 170 828 404 688 > $OUT/ncu_tile.log 2>&1
ncu -i /tmp/tile_full.ncu-rep --page raw --csv > $OUT/tile_raw.csv 2>/dev/null
ncu -i /tmp/tile_full.ncu-rep --page details --csv > $OUT/tile_details.csv 2>/dev/null
ncu -i /tmp/tile_full.ncu-rep --page source --csv --print-source sass -k regex:stage_tile -c 1 > $OUT/tile_source.csv 2>/dev/null

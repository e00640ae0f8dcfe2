#!/bin/bash
# Straight-line 3x3 window issue vs the rolled loop (normal and bare-MMA DBG builds).
OUT=gpurun_out/r02_sl
mkdir -p $OUT
for lib in "sl:paper_2410_23745_b200/libsyno.so:0" "nosl:gpu_lib/libsyno_nosl.so:0" "dbg_sl:gpu_lib/libsyno_dbg_sl.so:3072" "dbg_nosl:gpu_lib/libsyno_dbg.so:3072"; do
  IFS=: read name path dbg <<< "$lib"
  for env in "" "SYNO_TC_SMALL=0 SYNO_TC_G=1"; do
    echo "### $name env=[$env]" >> $OUT/res.txt
    env $env SYNO_LIB_PATH=$PWD/$path SYNO_TC_DEBUG=$dbg timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 10 2>&1 | grep "tc_gemm_fwd\|tc_gemm_dgrad" >> $OUT/res.txt
  done
done
for lib in "sl:paper_2410_23745_b200/libsyno.so" "nosl:gpu_lib/libsyno_nosl.so" "sl:paper_2410_23745_b200/libsyno.so" "nosl:gpu_lib/libsyno_nosl.so"; do
  IFS=: read name path <<< "$lib"
  SYNO_LIB_PATH=$PWD/$path timeout 300 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | grep "^{" | python -c "import json,sys;d=json.loads(sys.stdin.read());print('bench $name', d['ms_per_step'])" >> $OUT/res.txt
done
SYNO_LIB_PATH=$PWD/paper_2410_23745_b200/libsyno.so timeout 600 python -m pytest tests/test_gpu_tc.py -m gpu -q -x 2>&1 | tail -1 >> $OUT/res.txt

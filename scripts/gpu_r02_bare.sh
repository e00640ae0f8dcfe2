#!/bin/bash
# Bare MMA issue stream inside tc_gemm_kernel (DBG build, switches 1024|2048):
# is the conv3x3 64->64 @32 N=128 forward GEMM's per-MMA cost the kernel
# environment or its pipeline?  Library events per kernel class.
OUT=gpurun_out/r02_bare
mkdir -p $OUT
export SYNO_LIB_PATH=$PWD/gpu_lib/libsyno_dbg.so
for cfg in "0" "3072" "3104" "1024"; do
  for env in "" "SYNO_TC_SMALL=0 SYNO_TC_G=1"; do
    echo "### dbg=$cfg env=[$env]" >> $OUT/res.txt
    env $env SYNO_TC_DEBUG=$cfg timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 10 >> $OUT/res.txt 2>&1
  done
done

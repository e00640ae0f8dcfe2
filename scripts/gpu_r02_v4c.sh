#!/bin/bash
# chain_v4: single block vs four blocks (SYNO_TC_V4_ONE=0), PDL on / off (SYNO_NO_PDL), per-launch chain time.
OUT=gpurun_out/r02_v4c
mkdir -p $OUT
for L in "sep_shared 64 64 32 128" "conv3x3 64 64 32 128" "conv3x3 512 512 4 128"; do
  n=${L// /_}
  for cfg in "base:" "multi:SYNO_TC_V4_ONE=0" "old:SYNO_TC_NO_CHAIN_V4=1" "nopdl:SYNO_NO_PDL=1" "oldnopdl:SYNO_TC_NO_CHAIN_V4=1 SYNO_NO_PDL=1" "multinopdl:SYNO_TC_V4_ONE=0 SYNO_NO_PDL=1"; do
    tag=${cfg%%:*}; envs=${cfg#*:}
    env $envs timeout 300 python scripts/gemm_probe.py $L > $OUT/probe_${tag}_$n.log 2>&1
  done
done

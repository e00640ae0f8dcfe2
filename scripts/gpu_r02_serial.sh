#!/bin/bash
# Chain-rule launch time with the grad-weight on the caller's stream (SYNO_TC_SERIAL_BWD: no concurrent
# grad-input GEMM holding the SMs' registers / shared memory) vs the default concurrent backward.
OUT=gpurun_out/r02_serial
mkdir -p $OUT
for L in "sep_shared 64 64 32 128" "conv3x3 64 64 32 128" "sep_shared 512 512 4 128"; do
  n=${L// /_}
  for cfg in "conc:" "serial:SYNO_TC_SERIAL_BWD=1" "serialold:SYNO_TC_SERIAL_BWD=1 SYNO_TC_NO_CHAIN_V4=1" "concold:SYNO_TC_NO_CHAIN_V4=1" "wred:SYNO_TC_V4_WRED=1" "wred128:SYNO_TC_V4_WRED=1 SYNO_TC_V4_BLOCK=128" "b128:SYNO_TC_V4_BLOCK=128" "wred64:SYNO_TC_V4_WRED=1 SYNO_TC_V4_BLOCK=64"; do
    tag=${cfg%%:*}; envs=${cfg#*:}
    env $envs timeout 300 python scripts/gemm_probe.py $L > $OUT/probe_${tag}_$n.log 2>&1
  done
done
for cfg in "base:" "wred128:SYNO_TC_V4_WRED=1 SYNO_TC_V4_BLOCK=128" "b128:SYNO_TC_V4_BLOCK=128"; do
  tag=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 600 python bench.py --no-others --no-cpu-baseline > $OUT/bench_${tag}.log 2>&1
done

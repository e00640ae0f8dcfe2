#!/bin/bash
# A/B of environment switches on the ResNet-18 / ResNet-34 step (ms/step, 20 / 5 steps).
OUT=gpurun_out/${1:-ab}
mkdir -p $OUT
r18() { timeout 300 env "$@" python bench.py --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])"; }
for sw in ${SWS:-"X=0" "SYNO_TC_NO_BRES=1" "SYNO_TC_SERIAL_BWD=1" "SYNO_TC_WG_WAVES=2" "SYNO_TC_NO_PREP_FUSE=1" "SYNO_TC_DUAL_FOLD=1" "X=0"}; do
  echo "$sw $(r18 $sw)" >> $OUT/ab.txt
done
cat $OUT/ab.txt

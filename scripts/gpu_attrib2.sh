#!/bin/bash
OUT=gpurun_out/${1:-attrib2}
mkdir -p $OUT
for pdl in 0 1; do
for sk in "" chain "pack,fold,chain,cast,zero" gemm; do
  if [ $pdl = 1 ]; then export SYNO_NO_PDL=1; else unset SYNO_NO_PDL; fi
  echo "### nopdl=$pdl skip=$sk $(SYNO_SKIP=$sk timeout 300 python bench.py --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/attrib.txt
done; done

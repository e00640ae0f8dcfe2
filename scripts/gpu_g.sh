#!/bin/bash
OUT=gpurun_out/${1:-g}
mkdir -p $OUT
for g in 0 1 2 4; do
  echo "### G=$g" >> $OUT/g.txt
  SYNO_TC_G=$g timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 10 2>&1 | grep -E "fwd|dgrad" >> $OUT/g.txt
  SYNO_TC_G=$g timeout 120 python scripts/gemm_probe.py conv3x3 128 128 16 128 10 2>&1 | grep -E "fwd|dgrad" >> $OUT/g.txt
  echo "step $(SYNO_TC_G=$g timeout 300 python bench.py --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/g.txt
done

#!/bin/bash
OUT=gpurun_out/${1:-ks}
mkdir -p $OUT
for wv in 1; do
  echo "### waves=$wv" >> $OUT/ks.txt
  SYNO_TC_WG_WAVES=$wv timeout 120 python scripts/gemm_probe.py conv3x3 64 64 32 128 10 2>&1 | grep -E "wgrad|chain" >> $OUT/ks.txt
  SYNO_TC_WG_WAVES=$wv timeout 120 python scripts/gemm_probe.py conv3x3 512 512 4 128 10 2>&1 | grep -E "wgrad|chain" >> $OUT/ks.txt
  echo "step $(SYNO_TC_WG_WAVES=$wv timeout 300 python bench.py --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/ks.txt
  echo "skipchain $(SYNO_SKIP=chain SYNO_TC_WG_WAVES=$wv timeout 300 python bench.py --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/ks.txt
done

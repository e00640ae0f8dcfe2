#!/bin/bash
OUT=gpurun_out/${1:-t20}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for v in 0 1; do
  if [ $v = 1 ]; then export SYNO_TC_SERIAL_BWD=1; else unset SYNO_TC_SERIAL_BWD; fi
  echo "serial=$v r18 $(timeout 300 python bench.py --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/serial.txt
  echo "serial=$v r34 $(timeout 300 python bench.py --workload resnet34 --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/serial.txt
  echo "serial=$v qkv $(timeout 300 python bench.py --workload qkv --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'])")" >> $OUT/serial.txt
done

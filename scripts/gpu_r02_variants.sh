#!/bin/bash
# cfg4 sampled QKV variants (parity + bench) and the staged-engine preference (SYNO_TC_UNSTAGED=1 = off).
OUT=gpurun_out/r02_variants
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_qkv_variants.py tests/test_gpu_parity.py tests/test_gpu_tc.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py --workload qkv_variants > $OUT/bench_variants.log 2>&1
SYNO_TC_UNSTAGED=1 timeout 900 python bench.py --workload qkv_variants --no-cpu-baseline > $OUT/bench_variants_unstaged.log 2>&1
for r in 1 2; do
  timeout 900 python bench.py --workload sweep --no-cpu-baseline 2>/dev/null | grep "^{" > $OUT/sweep_staged_$r.json
  SYNO_TC_UNSTAGED=1 timeout 900 python bench.py --workload sweep --no-cpu-baseline 2>/dev/null | grep "^{" > $OUT/sweep_unstaged_$r.json
done

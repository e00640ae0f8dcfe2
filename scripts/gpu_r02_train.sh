#!/bin/bash
# Proxy training (cfg4): graph-captured step vs eager, loss parity of the two, the DP GPU tests.
OUT=gpurun_out/r02_train
mkdir -p $OUT
for i in 1 2; do
  timeout 600 python bench.py --workload qkv_train --no-cpu-baseline > $OUT/bench_graph_$i.log 2>&1
  timeout 600 python bench.py --workload qkv_train --no-cpu-baseline --no-graph > $OUT/bench_eager_$i.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -k "train or dp or proxy or autograd" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log

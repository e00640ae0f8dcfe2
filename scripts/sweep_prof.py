"""cProfile of one sweep pass (workers=1) over the first N corpus candidates:
where a candidate evaluation spends its host time.

    python scripts/sweep_prof.py [N]
"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_23745_b200 import pgraph as P  # noqa: E402
from paper_2410_23745_b200.sweep import run_shard  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
graphs, costs, fcap, pcap = bench.sweep_setup(n)
run_shard(graphs, range(len(graphs)), dtype=torch.float32, flops_cap=fcap, params_cap=pcap, workers=1)
torch.cuda.synchronize()
with P._CACHE_LOCK:
    P._CACHE.clear()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
recs, _ = run_shard(graphs, range(len(graphs)), dtype=torch.float32, flops_cap=fcap, params_cap=pcap, workers=1)
torch.cuda.synchronize()
pr.disable()
print(f"{len(graphs)} candidates in {time.perf_counter() - t0:.2f} s (workers=1)")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

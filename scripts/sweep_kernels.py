"""Per-kernel-class device time (library CUDA events) of one sweep pass
(workers=1) over the first N corpus candidates.

    python scripts/sweep_kernels.py [N]
"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_23745_b200 import _lib  # noqa: E402
from paper_2410_23745_b200 import pgraph as P  # noqa: E402
from paper_2410_23745_b200.sweep import run_shard  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
graphs, costs, fcap, pcap = bench.sweep_setup(n)
run_shard(graphs, range(len(graphs)), dtype=torch.float32, flops_cap=fcap, params_cap=pcap, workers=1)
torch.cuda.synchronize()
with P._CACHE_LOCK:
    P._CACHE.clear()
_lib.profile_begin()
t0 = time.perf_counter()
recs, _ = run_shard(graphs, range(len(graphs)), dtype=torch.float32, flops_cap=fcap, params_cap=pcap, workers=1)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
prof = _lib.profile_end()
print(f"{len(graphs)} candidates, {wall:.2f} s wall (workers=1)")
tot = sum(v["ms"] for v in prof.values())
print(f"library kernels: {tot:.1f} ms device time")
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])[:20]:
    print(f"  {k:26s} {v['launches']:6d} launches {v['ms']:9.1f} ms  {1e3 * v['ms'] / max(1, v['launches']):8.1f} us/launch")

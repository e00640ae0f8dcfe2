"""cProfile (all threads via sys.setprofile is too heavy: sample with
py-spy-like timing instead) -- wall time of one sweep pass at W workers and
the per-phase host time of `sweep.evaluate` (compile, inputs, forward,
backward, checks) summed over candidates.

    python scripts/sweep_prof_conc.py [workers]
"""
import sys
import threading
import time
from collections import defaultdict

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_23745_b200 import ops  # noqa: E402
from paper_2410_23745_b200 import pgraph as P  # noqa: E402
from paper_2410_23745_b200 import sweep as SW  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
graphs, costs, fcap, pcap = bench.sweep_setup(None)
order = SW.lpt_order(costs)
SW.run_dynamic(graphs, order, SW.LocalClaim(len(order)), dtype=torch.float32, flops_cap=fcap, params_cap=pcap,
               workers=W)
torch.cuda.synchronize()
with P._CACHE_LOCK:
    P._CACHE.clear()
acc = defaultdict(float)
lock = threading.Lock()
orig_hf, orig_f, orig_b = P.handle_for, ops.forward, ops.backward


def timed(name, fn):
    def w(*a, **k):
        t0 = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            with lock:
                acc[name] += time.perf_counter() - t0
    return w


SW_handle = timed("handle_for", orig_hf)
P.handle_for = SW_handle
ops.forward = timed("ops.forward (host)", orig_f)
ops.backward = timed("ops.backward (host)", orig_b)
t0 = time.perf_counter()
recs, _ = SW.run_dynamic(graphs, order, SW.LocalClaim(len(order)), dtype=torch.float32, flops_cap=fcap,
                         params_cap=pcap, workers=W)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(f"workers={W}: {len(recs)} candidates in {wall:.2f} s")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:24s} {v:8.3f} s (summed over threads)")

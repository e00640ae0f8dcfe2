"""Cold (fresh compile) evaluation of corpus candidates, as a sweep step runs
them: wall and event-timed device time per candidate, after a warm-up on
the batch-2 corpus (kernel modules loaded, pool primed).

    python scripts/sweep_cold.py 124 179 21 ...
"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2410_23745_b200 import workloads as WL  # noqa: E402
from paper_2410_23745_b200.sweep import evaluate  # noqa: E402

ids = [int(a) for a in sys.argv[1:]]
warm = WL.corpus(2)
for i in ids:
    evaluate(warm[i], i, i, dtype=torch.float32)
torch.cuda.synchronize()
graphs = WL.corpus(8)
tot_w = tot_d = 0.0
for i in ids:
    t0 = time.perf_counter()
    r = evaluate(graphs[i], i, i, dtype=torch.float32)
    torch.cuda.synchronize()
    w = time.perf_counter() - t0
    tot_w += w
    tot_d += r.seconds
    print(f"{i:5d} wall {w*1e3:9.2f} ms  device {r.seconds*1e3:9.2f} ms  {r.status}")
print(f"total wall {tot_w*1e3:.1f} ms device {tot_d*1e3:.1f} ms")

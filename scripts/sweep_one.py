"""Evaluate selected corpus candidates once (fp32, N=8) -- the target of
ncu captures of the universal-engine kernels.

    python scripts/sweep_one.py 170 828 404
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2410_23745_b200 import workloads as WL  # noqa: E402
from paper_2410_23745_b200.sweep import evaluate  # noqa: E402

graphs = WL.corpus(8)
for a in sys.argv[1:]:
    i = int(a)
    r = evaluate(graphs[i], i, i, dtype=torch.float32)
    torch.cuda.synchronize()
    print(r.line())
    print(r.diag())

"""Re-run chosen corpus candidates and print their evaluation records."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_23745_b200 import workloads as WL  # noqa: E402
from paper_2410_23745_b200.sweep import evaluate  # noqa: E402

ids = [int(a) for a in sys.argv[1:]]
graphs = WL.corpus(8)
for i in ids:
    r = evaluate(graphs[i], i, i, dtype=torch.float32)
    print(r.line())
    print(r.diag())

"""Per-kernel-class device time of single corpus candidates (fp32, N=8).

    python scripts/sweep_prof_one.py 124 179 21
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2410_23745_b200 import _lib, workloads as WL  # noqa: E402
from paper_2410_23745_b200.sweep import evaluate  # noqa: E402

graphs = WL.corpus(8)
for a in sys.argv[1:]:
    i = int(a)
    evaluate(graphs[i], i, i, dtype=torch.float32)  # warm: compile, tables, workspaces
    torch.cuda.synchronize()
    _lib.profile_begin()
    r = evaluate(graphs[i], i, i, dtype=torch.float32)
    torch.cuda.synchronize()
    prof = _lib.profile_end()
    print(r.line())
    print(r.diag())
    for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
        print(f"   {k:28s} {v['launches']:4d} launches {v['ms']:9.3f} ms")

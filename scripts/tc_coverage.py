"""Which cfg5 corpus candidates take a tensor-core path (host-side: handles
compile without a GPU).  Classes: in-budget candidates with weights, split by
weight rank -- a matrix weight (an output- or input-channel dim) makes the
contraction GEMM-shaped; vector weights only (a shared [K] tap vector) leave
a weighted window sum whose N = 1 contraction is gather-bound.

    python scripts/tc_coverage.py > profiles/r02_tc_coverage.txt
"""
import collections
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2410_23745_b200 import pgraph as P  # noqa: E402
from paper_2410_23745_b200.sweep import within_budget  # noqa: E402

PATH = {0: "universal engine", 1: "conv implicit GEMM", 2: "gathered GEMM"}
graphs, _, fcap, pcap = bench.sweep_setup()
cnt, fl = collections.Counter(), collections.Counter()
for g in graphs:
    h = P.handle_for(g)
    if not within_budget(h.flops_unstaged, h.params, fcap, pcap):
        key = ("over budget (not executed)", None)
    elif not h.w_shapes:
        key = ("no weights (window sums)", h.info.tc_path)
    else:
        key = ("matrix weight" if any(len(s) > 1 for s in h.w_shapes) else "vector weights only", h.info.tc_path)
    cnt[key] += 1
    fl[key] += h.flops_staged or h.flops_unstaged
print(f"cfg5 corpus, {len(graphs)} candidates (conv64 spec, N=8): tcgen05 path per class")
print(f"{'class':32s} {'path':20s} {'candidates':>10s} {'GFLOP (staged)':>15s}")
for k in sorted(cnt, key=lambda k: (k[0], -1 if k[1] is None else k[1])):
    print(f"{k[0]:32s} {PATH.get(k[1], '-'):20s} {cnt[k]:10d} {fl[k] / 1e9:15.1f}")
m_tc = sum(v for k, v in cnt.items() if k[0] == "matrix weight" and k[1])
m_all = sum(v for k, v in cnt.items() if k[0] == "matrix weight")
w_tc = sum(v for k, v in cnt.items() if k[0] in ("matrix weight", "vector weights only") and k[1])
w_all = sum(v for k, v in cnt.items() if k[0] in ("matrix weight", "vector weights only"))
print(f"\nmatrix-weight candidates on a tensor-core path: {m_tc}/{m_all}; all weighted: {w_tc}/{w_all}")

"""Count the corpus / QKV-variant stages that fall back to coordinate programs
(SYNO_PROG_LOG=1 prints them; this drives every candidate once, fp32)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2410_23745_b200 import workloads as WL  # noqa: E402
from paper_2410_23745_b200.sweep import evaluate  # noqa: E402

graphs = WL.corpus(8) if sys.argv[1] == "corpus" else [L.graph for L in WL.qkv_variants(2, 256)]
cap = 6039797760 if sys.argv[1] == "corpus" else None
for i, g in enumerate(graphs):
    evaluate(g, i, i, dtype=torch.float32, flops_cap=cap, params_cap=589824 if cap else None)
torch.cuda.synchronize()

"""Run one corpus candidate (fp32, N=8) and save y, dx, dws (for comparing
SYNO_NO_PERM=1 against the default in two processes).

    python scripts/perm_debug.py 331 out.pt
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2410_23745_b200 import ops, pgraph as P, workloads as WL  # noqa: E402

i = int(sys.argv[1])
g = WL.corpus(8)[i]
h = P.handle_for(g, None, True)
gen = torch.Generator(device="cuda").manual_seed(i)
x = torch.randn(h.x_shape, generator=gen, device="cuda")
ws = [torch.randn(s, generator=gen, device="cuda") for s in h.w_shapes]
dy = torch.randn(h.y_shape, generator=gen, device="cuda")
y = ops.forward(h, x, ws)
dx, dws = ops.backward(h, x, ws, dy)
torch.cuda.synchronize()
torch.save({"y": y.cpu(), "dx": dx.cpu(), "dws": [d.cpu() for d in dws]}, sys.argv[2])
print(h.describe())

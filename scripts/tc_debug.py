"""Debug driver for the tcgen05 path: one small conv, fwd then bwd, synced."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2410_23745_b200 import ops, pgraph as P, workloads as WL

op = sys.argv[1] if len(sys.argv) > 1 else "conv3x3"
L = WL.conv_layer("dbg", op, 64, 64, 8, 1)
h = P.handle_for(L.graph)
print("tc_path", h.info.tc_path, flush=True)
x = torch.randn(h.x_shape, device="cuda").bfloat16()
ws = [torch.randn(s, device="cuda").bfloat16() for s in h.w_shapes]
y = ops.forward(h, x, ws)
torch.cuda.synchronize()
print("fwd ok", float(y.float().abs().max()), flush=True)
import torch.nn.functional as F
ref = F.conv2d(x.float(), ws[0].float(), padding=1) if op == "conv3x3" else None
if ref is not None:
    print("fwd err", float((y.float() - ref).abs().max() / ref.abs().max()), flush=True)
dy = torch.randn(h.y_shape, device="cuda").bfloat16()
dx, dws = ops.backward(h, x, ws, dy)
torch.cuda.synchronize()
print("bwd ok", flush=True)

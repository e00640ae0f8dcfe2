"""Time one synthesized layer's forward and backward (CUDA events), for ncu runs.

    python scripts/layer_prof.py conv3x3 64 64 32 128 [iters]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_23745_b200 import ops, pgraph as P, workloads as WL  # noqa: E402

op, cin, cout, h, batch = sys.argv[1], *map(int, sys.argv[2:6])
iters = int(sys.argv[6]) if len(sys.argv) > 6 else 5
L = WL.conv_layer("p", op, cin, cout, h, batch)
hd = P.handle_for(L.graph)
x = torch.randn(hd.x_shape, device="cuda").bfloat16()
ws = [torch.randn(s, device="cuda").bfloat16() for s in hd.w_shapes]
dy = torch.randn(hd.y_shape, device="cuda").bfloat16()
for _ in range(2):
    ops.forward(hd, x, ws)
    ops.backward(hd, x, ws, dy)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record()
for _ in range(iters):
    ops.forward(hd, x, ws)
e[1].record()
for _ in range(iters):
    ops.backward(hd, x, ws, dy)
e[2].record()
torch.cuda.synchronize()
f = e[0].elapsed_time(e[1]) / iters
b = e[1].elapsed_time(e[2]) / iters
print(f"{op} {cin}->{cout} @{h} N={batch}: fwd {f*1e3:.1f} us  bwd {b*1e3:.1f} us  "
      f"({hd.flops_staged/1e9:.2f} GFLOP fwd; {hd.flops_staged/(f*1e-3)/1e12:.1f} TF/s fwd, "
      f"{2*hd.flops_staged/(b*1e-3)/1e12:.1f} TF/s bwd)")

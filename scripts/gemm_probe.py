"""Per-kernel-class device time of one layer's fwd + bwd (library CUDA events).

    python scripts/gemm_probe.py op c_in c_out h batch [iters] [dtype]
Env SYNO_TC_DEBUG (1 skip epilogue stores, 2 skip MMAs, 4 skip A loads,
8 skip B loads) and SYNO_TC_TRACE are read by the library."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_23745_b200 import _lib, ops, pgraph as P, workloads as WL  # noqa: E402

op, cin, cout, h, batch = sys.argv[1], *map(int, sys.argv[2:6])
iters = int(sys.argv[6]) if len(sys.argv) > 6 else 10
dt = getattr(torch, sys.argv[7]) if len(sys.argv) > 7 else torch.bfloat16
L = WL.qkv(batch) if op == "qkv" else WL.conv_layer("p", op, cin, cout, h, batch)
hd = P.handle_for(L.graph)
x = torch.randn(hd.x_shape, device="cuda").to(dt)
ws = [torch.randn(s, device="cuda").to(dt) for s in hd.w_shapes]
dy = torch.randn(hd.y_shape, device="cuda").to(dt)
for _ in range(2):
    ops.forward(hd, x, ws)
    ops.backward(hd, x, ws, dy)
torch.cuda.synchronize()
_lib.profile_begin()
for _ in range(iters):
    ops.forward(hd, x, ws)
    ops.backward(hd, x, ws, dy)
torch.cuda.synchronize()
prof = _lib.profile_end()
F = hd.flops_unstaged
print(f"{op} {cin}->{cout} @{h} N={batch} {dt} ({F/1e9:.2f} GFLOP per GEMM)")
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    per = v["ms"] / v["launches"] * 1e3
    extra = f" {v['flops']/v['launches']/(per*1e-6)/1e12:7.1f} TF/s" if v["flops"] else ""
    extra += f" {v['bytes']/v['launches']/(per*1e-6)/1e9:7.1f} GB/s" if v["bytes"] else ""
    print(f"  {k:22s} {v['launches']/iters:4.1f}/iter {per:9.2f} us/launch{extra}")

"""GPU: the tcgen05 contraction path (bf16) on the config operator family at
real layer sizes, against a plain PyTorch fp32 reference of the same op
(conv2d / matmul on the bf16-rounded inputs, autograd for the gradients),
tolerance 2e-2 rel (max|d| / max|want|, reference test_codegen.py:95-97)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel(got, want):
    got = got.double()
    want = want.double()
    return float((got - want).abs().max() / max(float(want.abs().max()), 1e-12))


def _layer(op, c_in, c_out, h, batch):
    from paper_2410_23745_b200 import workloads as WL
    return WL.conv_layer("t", op, c_in, c_out, h, batch)


def _torch_ref(op, x, ws, c_in, c_out):
    import torch
    import torch.nn.functional as F
    if op == "conv3x3":
        return F.conv2d(x, ws[0], padding=1)
    if op == "conv3x3_s2":
        return F.conv2d(x, ws[0], stride=2, padding=1)
    if op == "shortcut_s2":
        return F.conv2d(x, ws[0], stride=2, padding=0)
    if op == "pointwise":
        return F.conv2d(x, ws[0][:, :, None, None])
    if op == "sep_shared":
        w = ws[0][:, :, :, None] * ws[1][None, None, None, :]  # [co, ci, kh] x [kw]
        return F.conv2d(x, w, padding=1)
    raise ValueError(op)


CASES = [
    ("conv3x3", 64, 64, 32, 2),
    ("conv3x3", 3, 64, 32, 2),       # stem: C_in padded to 8, K tail zero-filled by TMA
    ("conv3x3", 8, 64, 32, 2),       # one 16-wide K step per window (kq_last), no padding
    ("conv3x3", 64, 128, 16, 3),
    ("conv3x3", 128, 256, 8, 2),
    ("conv3x3", 256, 512, 4, 2),
    ("conv3x3", 64, 64, 7, 3),       # 7x7 maps (ResNet-34 stage 4 shape)
    ("conv3x3_s2", 64, 128, 16, 2),
    ("conv3x3_s2", 128, 256, 8, 2),
    ("shortcut_s2", 64, 128, 16, 2),
    ("sep_shared", 64, 64, 32, 2),
    ("pointwise", 64, 128, 32, 2),
    # BN = 256 with many M tiles: the CTA-pair (cta_group::2) configuration
    ("conv3x3", 256, 256, 14, 8),
    ("conv3x3_s2", 128, 256, 14, 8),
    ("conv3x3", 512, 512, 7, 16),
]


@pytest.mark.parametrize("op,c_in,c_out,h,batch", CASES)
def test_tc_conv_family_fwd_bwd(cuda, op, c_in, c_out, h, batch):
    import torch
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    L = _layer(op, c_in, c_out, h, batch)
    hd = P.handle_for(L.graph)
    assert hd.info.tc_path == 1
    g = torch.Generator(device="cpu").manual_seed(3)
    x = torch.randn(hd.x_shape, generator=g).to("cuda", torch.bfloat16)
    ws = [(torch.randn(s, generator=g) * 0.2).to("cuda", torch.bfloat16) for s in hd.w_shapes]
    dy = torch.randn(hd.y_shape, generator=g).to("cuda", torch.bfloat16)
    y = ops.forward(hd, x, ws)
    dx, dws = ops.backward(hd, x, ws, dy)
    torch.cuda.synchronize()
    xf = x.float().requires_grad_(True)
    wf = [w.float().requires_grad_(True) for w in ws]
    yr = _torch_ref(op, xf, wf, c_in, c_out)
    assert yr.shape == y.shape
    assert _rel(y, yr) < 2e-2
    yr.backward(dy.float())
    assert _rel(dx, xf.grad) < 2e-2
    for a, b in zip(dws, wf):
        assert _rel(a, b.grad) < 2e-2


@pytest.mark.parametrize("batch,t", [(2, 256), (4, 512)])  # (4, 512): CTA-pair forward / grad-input
def test_tc_qkv_projection(cuda, batch, t):
    import torch
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    from paper_2410_23745_b200 import workloads as WL
    L = WL.qkv(batch=batch, t=t)
    hd = P.handle_for(L.graph)
    assert hd.info.tc_path == 1
    g = torch.Generator(device="cpu").manual_seed(4)
    x = torch.randn(hd.x_shape, generator=g).to("cuda", torch.bfloat16)
    w = (torch.randn(hd.w_shapes[0], generator=g) * 0.05).to("cuda", torch.bfloat16)
    dy = torch.randn(hd.y_shape, generator=g).to("cuda", torch.bfloat16)
    y = ops.forward(hd, x, [w])
    dx, (dw,) = ops.backward(hd, x, [w], dy)
    xf = x.float().requires_grad_(True)
    wf = w.float().requires_grad_(True)
    yr = xf @ wf.t()
    yr.backward(dy.float())
    assert _rel(y, yr) < 2e-2
    assert _rel(dx, xf.grad) < 2e-2
    assert _rel(dw, wf.grad) < 2e-2


def test_tc_qkv_projection_fp32_pair(cuda):
    """fp32 through the split-bf16 path on the CTA-pair configuration
    (forward, grad-input and grad-weight all BN = 256 with several M tiles),
    against torch float64, tolerance 1e-4 rel."""
    import torch
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    from paper_2410_23745_b200 import workloads as WL
    L = WL.qkv(batch=4, t=512)
    hd = P.handle_for(L.graph)
    g = torch.Generator(device="cpu").manual_seed(5)
    x = torch.randn(hd.x_shape, generator=g).to("cuda")
    w = (torch.randn(hd.w_shapes[0], generator=g) * 0.05).to("cuda")
    dy = torch.randn(hd.y_shape, generator=g).to("cuda")
    y = ops.forward(hd, x, [w])
    dx, (dw,) = ops.backward(hd, x, [w], dy)
    xd = x.double().requires_grad_(True)
    wd = w.double().requires_grad_(True)
    yr = xd @ wd.t()
    yr.backward(dy.double())
    assert _rel(y, yr) < 1e-4
    assert _rel(dx, xd.grad) < 1e-4
    assert _rel(dw, wd.grad) < 1e-4


@pytest.mark.parametrize("op,c_in,c_out,h,batch", [("conv3x3", 64, 64, 16, 2), ("sep_shared", 64, 64, 16, 2),
                                                   ("conv3x3_s2", 64, 128, 8, 2)])
@pytest.mark.parametrize("dtype", ["bfloat16", "float32"])
def test_backward_reuse_flags_match(cuda, op, c_in, c_out, h, batch, dtype):
    """syno_backward_ex(X_UNCHANGED | W_UNCHANGED) reuses the forward's packed x
    and grad-input weight operand; results equal the flag-free backward."""
    import torch
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    dt = getattr(torch, dtype)
    L = _layer(op, c_in, c_out, h, batch)
    hd = P.handle_for(L.graph)
    g = torch.Generator(device="cpu").manual_seed(5)
    x = torch.randn(hd.x_shape, generator=g).to("cuda", dt)
    ws = [(torch.randn(s, generator=g) * 0.2).to("cuda", dt) for s in hd.w_shapes]
    dy = torch.randn(hd.y_shape, generator=g).to("cuda", dt)
    dx0, dw0 = ops.backward(hd, x, ws, dy)
    ops.forward(hd, x, ws)
    dx1, dw1 = ops.backward(hd, x, ws, dy, x_unchanged=True, w_unchanged=True)
    torch.cuda.synchronize()
    # split-K partial sums are combined with fp32 atomics (order not fixed)
    assert _rel(dx1, dx0) < 1e-6
    for a, b in zip(dw0, dw1):
        assert _rel(a, b) < 1e-6


@pytest.mark.parametrize("want", [(True, True), (True, False), (False, True)], ids=["both", "w0", "w1"])
@pytest.mark.parametrize("dtype", ["bfloat16", "float32"])
def test_sep_shared_weight_gradient_subsets(cuda, want, dtype):
    """sep_shared's [K] weight takes its gradient from the main weight's chain
    pass (side output, block partials combined by the last block); any subset
    of weight gradients, called repeatedly (dWf and the block counter are left
    zeroed for the next call), matches autograd."""
    import torch
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    dt = getattr(torch, dtype)
    L = _layer("sep_shared", 128, 128, 16, 2)
    hd = P.handle_for(L.graph)
    g = torch.Generator(device="cpu").manual_seed(6)
    x = torch.randn(hd.x_shape, generator=g).to("cuda", dt)
    ws = [(torch.randn(s, generator=g) * 0.2).to("cuda", dt) for s in hd.w_shapes]
    # float64 reference (a float32 torch conv may run in TF32)
    xf = x.double().requires_grad_(True)
    wf = [w.double().requires_grad_(True) for w in ws]
    yr = _torch_ref("sep_shared", xf, wf, 128, 128)
    for it in range(3):
        dy = torch.randn(hd.y_shape, generator=g).to("cuda", dt)
        _, dws = ops.backward(hd, x, ws, dy, want_dx=False, want_dw=list(want))
        torch.cuda.synchronize()
        refs = torch.autograd.grad(yr, wf, dy.double(), retain_graph=True)
        tol = 2e-2 if dtype == "bfloat16" else 1e-4
        for j in range(2):
            if want[j]:
                assert _rel(dws[j], refs[j]) < tol, (it, j)
            else:
                assert dws[j] is None

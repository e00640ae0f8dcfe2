"""GPU parity at the EXACT timed configurations of bench.py.

Every distinct layer of the ResNet-18 step (N=128) and of the ResNet-34 step
(N=256), and the QKV projection at B=16, T=1024, run through the same
handles, the same call sequence (forward, then syno_backward_ex with the
X_UNCHANGED | W_UNCHANGED training-step flags) and therefore the same kernel
configurations as the benchmark: the two-wave split-K grad-weight, the
odd-tail CTA-pair staging, the two-CTA-per-SM small-tile GEMMs and the
in-place QKV weight.  References:

* y and dx: torch float64 on a slice of the batch (images are independent,
  reference codegen.py:626-630), bf16-rounded inputs upcast;
* dW: the full batch (dW sums over it, codegen.py:728-742) with torch
  float32 convolutions/matmuls, TF32 disabled (relative error ~1e-6, far
  below the bf16 tolerance).

Tolerance bf16 2e-2 rel, max|d| / max|want| (reference test_codegen.py:95-97).
"""
from __future__ import annotations

import math

import pytest

pytestmark = pytest.mark.gpu

TOL = 2e-2
SLICE = 4


def _rel(got, want):
    got = got.double()
    want = want.double()
    return float((got - want).abs().max() / max(float(want.abs().max()), 1e-12))


def _conv_ref(op, x, ws):
    import torch.nn.functional as F
    if op == "conv3x3":
        return F.conv2d(x, ws[0], padding=1)
    if op == "conv3x3_s2":
        return F.conv2d(x, ws[0], stride=2, padding=1)
    if op == "shortcut_s2":
        return F.conv2d(x, ws[0], stride=2, padding=0)
    if op == "sep_shared":
        return F.conv2d(x, ws[0][:, :, :, None] * ws[1][None, None, None, :], padding=1)
    raise ValueError(op)


def _distinct(rows):
    seen, out = set(), []
    for name, op, ci, co, h in rows:
        if (op, ci, co, h) not in seen:
            seen.add((op, ci, co, h))
            out.append((name, op, ci, co, h))
    return out


def _run_bench_sequence(hd, x, ws, dy):
    """bench.py's call sequence: forward, then the flagged backward."""
    from paper_2410_23745_b200 import ops
    y = ops.forward(hd, x, ws)
    dx, dws = ops.backward(hd, x, ws, dy, x_unchanged=True, w_unchanged=True)
    return y, dx, dws


def _check_conv_layer(op, ci, co, h, batch, seed):
    import torch

    from paper_2410_23745_b200 import pgraph as P
    from paper_2410_23745_b200 import workloads as WL
    L = WL.conv_layer("b", op, ci, co, h, batch)
    hd = P.handle_for(L.graph)
    assert hd.info.tc_path == 1
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(hd.x_shape, generator=g, device="cuda").bfloat16()
    ws = [(torch.randn(s, generator=g, device="cuda") / math.sqrt(max(1, math.prod(s[1:])))).bfloat16()
          for s in hd.w_shapes]
    dy = torch.randn(hd.y_shape, generator=g, device="cuda").bfloat16()
    y, dx, dws = _run_bench_sequence(hd, x, ws, dy)
    torch.cuda.synchronize()
    # y, dx on a batch slice in float64
    xs = x[:SLICE].double().requires_grad_(True)
    wd = [w.double() for w in ws]
    ys = _conv_ref(op, xs, wd)
    ys.backward(dy[:SLICE].double())
    assert _rel(y[:SLICE], ys) < TOL, "y"
    assert _rel(dx[:SLICE], xs.grad) < TOL, "dx"
    # the LAST images too: the tail M tiles / odd split-K tail
    xt = x[-SLICE:].double().requires_grad_(True)
    yt = _conv_ref(op, xt, wd)
    yt.backward(dy[-SLICE:].double())
    assert _rel(y[-SLICE:], yt) < TOL, "y tail"
    assert _rel(dx[-SLICE:], xt.grad) < TOL, "dx tail"
    # dW over the full batch, float32 without TF32
    prev = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False
    try:
        wf = [w.float().requires_grad_(True) for w in ws]
        yf = _conv_ref(op, x.float(), wf)
        grads = torch.autograd.grad(yf, wf, dy.float())
    finally:
        torch.backends.cudnn.allow_tf32 = prev
    for j, (a, b) in enumerate(zip(dws, grads)):
        assert _rel(a, b) < TOL, f"dw{j}"


def _r18():
    from paper_2410_23745_b200.configs import resnet18_table
    return _distinct(resnet18_table())


def _r34():
    from paper_2410_23745_b200.configs import resnet34_table
    return _distinct(resnet34_table())


@pytest.mark.parametrize("name,op,ci,co,h", _r18(), ids=[r[0] for r in _r18()])
def test_resnet18_layer_at_bench_batch(cuda, name, op, ci, co, h):
    _check_conv_layer(op, ci, co, h, 128, seed=11)


@pytest.mark.parametrize("name,op,ci,co,h", _r34(), ids=[r[0] for r in _r34()])
def test_resnet34_layer_at_bench_batch(cuda, name, op, ci, co, h):
    _check_conv_layer(op, ci, co, h, 256, seed=12)


def _check_qkv(batch, t, e, e3, seed):
    import torch

    from paper_2410_23745_b200 import pgraph as P
    from paper_2410_23745_b200 import workloads as WL
    L = WL.qkv(batch=batch, t=t, e=e, e3=e3)
    hd = P.handle_for(L.graph)
    assert hd.info.tc_path == 1
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(hd.x_shape, generator=g, device="cuda").bfloat16()
    w = (torch.randn(hd.w_shapes[0], generator=g, device="cuda") / math.sqrt(e)).bfloat16()
    dy = torch.randn(hd.y_shape, generator=g, device="cuda").bfloat16()
    y, dx, (dw,) = _run_bench_sequence(hd, x, [w], dy)
    torch.cuda.synchronize()
    wd = w.double()
    for sl in (slice(0, 2), slice(batch - 2, batch)):
        xs = x[sl].double()
        assert _rel(y[sl], xs @ wd.t()) < TOL, "y"
        assert _rel(dx[sl], dy[sl].double() @ wd) < TOL, "dx"
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        dwr = dy.float().reshape(-1, e3).t() @ x.float().reshape(-1, e)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    assert _rel(dw, dwr) < TOL, "dw"


def test_qkv_at_bench_shape(cuda):
    """B=16, T=1024, E=768, E3=2304: the bench's QKV workload and one layer
    of the proxy-training step."""
    _check_qkv(16, 1024, 768, 2304, seed=13)


@pytest.mark.parametrize("e", [96, 128, 200])
def test_qkv_in_place_weight_odd_widths(cuda, e):
    """The in-place [N][C] weight read (forward K-major, grad-input MN-major)
    at C not a multiple of 64 (partly / fully out-of-bounds 64-wide loads)
    and at BN = 128 (two CTAs per SM)."""
    _check_qkv(2, 256, e, 3 * e, seed=14)


@pytest.mark.parametrize("ci,co", [(96, 96), (200, 128), (128, 200)])
def test_pointwise_odd_widths(cuda, ci, co):
    import torch

    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    from paper_2410_23745_b200 import workloads as WL
    from paper_2410_23745_b200.pgraph import build_spec, parse_steps
    ref = {"C_out": co, "C_in": ci, "H": 16, "W": 16, "N": 4}
    spec = build_spec("pw", ("C_out", "C_in", "H", "W", "N"), (), ref, ("C_out", "H", "W"), ("C_in", "H", "W"),
                      ("N",))
    hd = P.handle_for(parse_steps(WL.POINTWISE, spec))
    g = torch.Generator(device="cuda").manual_seed(15)
    x = torch.randn(hd.x_shape, generator=g, device="cuda").bfloat16()
    w = (torch.randn(hd.w_shapes[0], generator=g, device="cuda") / math.sqrt(ci)).bfloat16()
    dy = torch.randn(hd.y_shape, generator=g, device="cuda").bfloat16()
    y = ops.forward(hd, x, [w])
    dx, (dw,) = ops.backward(hd, x, [w], dy, x_unchanged=True, w_unchanged=True)
    xd, wd, dyd = x.double(), w.double(), dy.double()
    yr = torch.einsum("oc,nchw->nohw", wd, xd)
    assert _rel(y, yr) < TOL
    assert _rel(dx, torch.einsum("oc,nohw->nchw", wd, dyd)) < TOL
    assert _rel(dw, torch.einsum("nohw,nchw->oc", dyd, xd)) < TOL

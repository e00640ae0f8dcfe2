"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden outputs and the pinned CPU oracle.

Tolerances (metric rel_err = max|d| / max|want|,
reference test_codegen.py:95-97): integer index maps bit-exact;
float64 1e-10; float32 1e-4; bfloat16 2e-2 (oracle fed bf16-rounded inputs).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import CASE_IDS, CASES, GOLDEN, case_tensors

from oracle import nest_oracle as O

pytestmark = pytest.mark.gpu

TOL = {"float64": 1e-10, "float32": 1e-4, "bfloat16": 2e-2}


def _torch():
    import torch
    return torch


def _run(case, x, ws, up, dtype, staged=False):
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    torch = _torch()
    g = P.parse_operator(case["document"])
    h = P.handle_for(g, case["assignment"], staged)
    xd = ops.to_device(x, dtype)
    wd = [ops.to_device(w, dtype) for w in ws]
    ud = ops.to_device(up, dtype)
    y = ops.forward(h, xd, wd)
    dx, dws = ops.backward(h, xd, wd, ud, True, True)
    torch.cuda.synchronize()
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    return f(y), f(dx), [f(d) for d in dws]


def _rounded(a, dtype):
    torch = _torch()
    return torch.from_numpy(np.asarray(a)).to(getattr(torch, dtype)).double().numpy()


@pytest.mark.parametrize("dtype", ["float64", "float32", "bfloat16"])
@pytest.mark.parametrize("case", CASES, ids=CASE_IDS)
def test_golden_forward_backward(cuda, case, dtype):
    x, ws, up, y, ys, dws = case_tensors(case)
    env, bs = case["env"], case["batch_shape"]
    if dtype != "float64":
        x, up = _rounded(x, dtype), _rounded(up, dtype)
        ws = [_rounded(w, dtype) for w in ws]
        y = O.interpret(case["nest"], env, x, ws, bs)
        dws = O.weight_gradient(case["nest"], env, x, up, ws, bs) if ws else []
    dx_want = O.input_gradient(case["nest"], env, x, up, ws, bs)
    gy, gdx, gdw = _run(case, x, ws, up, dtype)
    tol = TOL[dtype]
    assert O.rel_err(gy, y) < tol
    assert O.rel_err(gdx, dx_want) < tol
    for a, b in zip(gdw, dws):
        assert O.rel_err(a, b) < tol
    if dtype == "float64":
        gys, _, _ = _run(case, x, ws, up, dtype, staged=True)
        assert O.rel_err(gys, ys) < tol


@pytest.mark.parametrize("case", CASES, ids=CASE_IDS)
def test_index_maps_bit_exact(cuda, case):
    """K1 tables evaluate every coordinate exactly like codegen._eval_array."""
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    g = P.parse_operator(case["document"])
    h = P.handle_for(g, case["assignment"])
    nest = O.parse_nest(case["nest"], case["env"])
    for t, term in enumerate(nest.stages[0].terms):
        for c in range(len(term.exprs)):
            got = ops.index_map(h, t, c).cpu().numpy()
            want = O.index_values(case["nest"], case["env"], t, c, case["batch_shape"]).reshape(-1)
            assert np.array_equal(got, want), (t, c)


def _corpus():
    ops_ = [ln.strip() for ln in open(os.path.join(GOLDEN, "corpus_conv64.txt")) if ln.strip()]
    return ops_


CORPUS_SPEC = dict(name="conv64", primaries=("C_out", "C_in", "H", "W", "N"), coeffs=("K", "s"),
                   reference={"C_out": 64, "C_in": 64, "H": 32, "W": 32, "K": 3, "s": 2, "N": 8},
                   output=("C_out", "H", "W"), input_=("C_in", "H", "W"), batch=("N",))
REDUCED = [
    {"C_out": 4, "C_in": 4, "H": 4, "W": 4, "K": 3, "s": 2, "N": 2},
    {"C_out": 2, "C_in": 4, "H": 8, "W": 4, "K": 3, "s": 2, "N": 2},
    {"C_out": 4, "C_in": 2, "H": 4, "W": 8, "K": 3, "s": 2, "N": 2},
    {"C_out": 2, "C_in": 2, "H": 4, "W": 4, "K": 3, "s": 2, "N": 2},
]


def reduced_case(op):
    from paper_2410_23745_b200 import codegen as C
    from paper_2410_23745_b200 import pgraph as P
    spec = P.build_spec(**CORPUS_SPEC)
    g = P.parse_steps(op, spec)
    for red in REDUCED:
        try:
            if C.flops(g, red) * 4 > 2e7:
                continue
            return g, red
        except Exception:
            continue
    return g, None


@pytest.mark.parametrize("chunk", range(8))
def test_corpus_reduced_fp32(cuda, chunk):
    """Every 8th corpus operator per chunk, at a reduced assignment, fwd + bwd in fp32."""
    from paper_2410_23745_b200 import codegen as C
    from paper_2410_23745_b200 import pgraph as P
    ops_ = _corpus()[chunk::8]
    checked = 0
    for op in ops_:
        g, red = reduced_case(op)
        if red is None:
            continue
        h = P.handle_for(g, red)
        text = C.emit_loop_nest(g, red)
        rng = np.random.default_rng(checked)
        x = rng.standard_normal(h.x_shape)
        ws = [rng.standard_normal(s) for s in h.w_shapes]
        up = rng.standard_normal(h.y_shape)
        xr, upr = _rounded(x, "float32"), _rounded(up, "float32")
        wr = [_rounded(w, "float32") for w in ws]
        case = {"document": g.document, "assignment": red}
        gy, gdx, gdw = _run(case, xr, wr, upr, "float32")
        bs = h.x_shape[:1]
        assert O.rel_err(gy, O.interpret(text, red, xr, wr, bs)) < 1e-4, op
        assert O.rel_err(gdx, O.input_gradient(text, red, xr, upr, wr, bs)) < 1e-4, op
        for a, b in zip(gdw, O.weight_gradient(text, red, xr, upr, wr, bs) if wr else []):
            assert O.rel_err(a, b) < 1e-4, op
        checked += 1
    assert checked >= len(ops_) // 2


def test_cfg1_full_size_fp32(cuda):
    """cfg1: conv3x3 N=8 C=64 H=W=32 fp32 forward vs the oracle at full size."""
    from paper_2410_23745_b200 import codegen as C
    from paper_2410_23745_b200 import pgraph as P
    case = next(c for c in CASES if c["name"] == "cfg1_reduced")
    g = P.parse_operator(case["document"])
    h = P.handle_for(g)
    rng = np.random.default_rng(0)
    x = _rounded(rng.standard_normal(h.x_shape), "float32")
    w = _rounded(rng.standard_normal(h.w_shapes[0]), "float32")
    text = C.emit_loop_nest(g)
    env = dict(g.spec.reference)
    gy, _, _ = _run({"document": g.document, "assignment": None}, x, [w], np.zeros(h.y_shape), "float32")
    want = O.interpret(text, env, x, [w], (8,))
    assert O.rel_err(gy, want) < 1e-4


def test_numpy_shims_match_reference_signatures(cuda):
    """interpret / weight_gradient with numpy in, numpy float64 out (codegen.py:598, 664)."""
    from paper_2410_23745_b200 import codegen as C
    from paper_2410_23745_b200 import pgraph as P
    from paper_2410_23745_b200.errors import ShapeMismatch
    case = next(c for c in CASES if c["name"] == "conv2d_8")
    x, ws, up, y, ys, dws = case_tensors(case)
    g = P.parse_operator(case["document"])
    out = C.interpret(g, x, ws)
    assert isinstance(out, np.ndarray) and out.dtype == np.float64
    assert O.rel_err(out, y) < 1e-12
    assert O.rel_err(C.interpret(g, x, ws, staged=True), ys) < 1e-12
    (dw,) = C.weight_gradient(g, x, up, ws)
    assert O.rel_err(dw, dws[0]) < 1e-12
    with pytest.raises(ShapeMismatch):
        C.interpret(g, x.transpose(1, 0, 2).copy()[:, :, :7], ws)
    with pytest.raises(ShapeMismatch):
        C.interpret(g, x)
    with pytest.raises(ShapeMismatch):
        C.interpret(g, x, [np.zeros((8, 8, 3, 2))])


def test_torch_autograd_module(cuda):
    torch = _torch()
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    case = next(c for c in CASES if c["name"] == "sep_shared")
    g = P.parse_operator(case["document"])
    m = ops.SynoOperator(g, dtype=torch.float64)
    x = torch.randn(m.h.x_shape, dtype=torch.float64, device="cuda", requires_grad=True)
    assert torch.autograd.gradcheck(lambda a, *w: ops.SynoFunction.apply(m.h, a, *w), (x, *m.weight),
                                    eps=1e-6, atol=1e-7)


@pytest.mark.parametrize("name", ["conv2d_8", "strided_conv1d", "sep_shared", "bpool", "corpus0003", "corpus0011"])
def test_program_fallback_matches_oracle(cuda, name, monkeypatch):
    """Stages whose index tables exceed the budget evaluate coordinate programs
    on the fly; SYNO_TABLE_LIMIT=2 forces that path on golden cases."""
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    torch = _torch()
    case = next(c for c in CASES if c["name"] == name)
    monkeypatch.setenv("SYNO_TABLE_LIMIT", "2")
    h = P.Handle(case["document"], case["assignment"], False)  # uncached: a fresh device plan
    x, ws, up, y, _, dws = case_tensors(case)
    xd = ops.to_device(x, "float64")
    wd = [ops.to_device(w, "float64") for w in ws]
    ud = ops.to_device(up, "float64")
    gy = ops.forward(h, xd, wd)
    gdx, gdw = ops.backward(h, xd, wd, ud)
    torch.cuda.synchronize()
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    env, bs = case["env"], case["batch_shape"]
    assert O.rel_err(f(gy), y) < 1e-10
    assert O.rel_err(f(gdx), O.input_gradient(case["nest"], env, x, up, ws, bs)) < 1e-10
    for a, b in zip(gdw, dws):
        assert O.rel_err(f(a), b) < 1e-10


def test_cli_eval_against_reference_golden(cuda, tmp_path):
    """`python -m paper_2410_23745_b200 eval` on tensors in the
    reference's file format, compared with the reference's own outputs."""
    import subprocess
    import sys

    from paper_2410_23745_b200.codegen import load_tensor, save_tensor
    from conftest import ROOT
    case = next(c for c in CASES if c["name"] == "sep_shared")
    x, ws, up, y, _, dws = case_tensors(case)
    (tmp_path / "op.txt").write_text(case["document"])
    save_tensor(tmp_path / "x.tensor", x)
    save_tensor(tmp_path / "up.tensor", up)
    wpaths = []
    for j, w in enumerate(ws):
        save_tensor(tmp_path / f"w{j}.tensor", w)
        wpaths.append(str(tmp_path / f"w{j}.tensor"))
    gpaths = [str(tmp_path / f"dw{j}.tensor") for j in range(len(ws))]
    cmd = [sys.executable, "-m", "paper_2410_23745_b200", "eval", "--op", str(tmp_path / "op.txt"),
           "--input", str(tmp_path / "x.tensor"), "--weights", *wpaths, "--output", str(tmp_path / "y.tensor"),
           "--upstream", str(tmp_path / "up.tensor"), "--grad-input", str(tmp_path / "dx.tensor"),
           "--grad-weights", *gpaths]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert O.rel_err(load_tensor(tmp_path / "y.tensor"), y) < 1e-10
    for p, want in zip(gpaths, dws):
        assert O.rel_err(load_tensor(p), want) < 1e-10
    dx_want = O.input_gradient(case["nest"], case["env"], x, up, ws, case["batch_shape"])
    assert O.rel_err(load_tensor(tmp_path / "dx.tensor"), dx_want) < 1e-10


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("case", CASES, ids=CASE_IDS)
def test_staged_handles_forward_backward(cuda, case, dtype):
    """SYNO_STAGED handles run the rfactored nest forward and, where every
    tensor is read once, reverse-mode through its stages backward; the math
    is the unstaged operator's (reference weight_gradient differentiates the
    unstaged nest, codegen.py:680), so the same oracle values apply."""
    x, ws, up, y, ys, dws = case_tensors(case)
    env, bs = case["env"], case["batch_shape"]
    if dtype != "float64":
        x, up = _rounded(x, dtype), _rounded(up, dtype)
        ws = [_rounded(w, dtype) for w in ws]
        y = O.interpret(case["nest"], env, x, ws, bs)
        dws = O.weight_gradient(case["nest"], env, x, up, ws, bs) if ws else []
    dx_want = O.input_gradient(case["nest"], env, x, up, ws, bs)
    gy, gdx, gdw = _run(case, x, ws, up, dtype, staged=True)
    tol = TOL[dtype]
    assert O.rel_err(gy, y) < tol
    assert O.rel_err(gdx, dx_want) < tol
    for a, b in zip(gdw, dws):
        assert O.rel_err(a, b) < tol


@pytest.mark.parametrize("chunk", range(8))
def test_corpus_reduced_staged_fp32(cuda, chunk):
    """Every corpus operator (all 1024 over the 8 chunks) through staged
    handles (rfactored forward, staged backward where it applies) at reduced
    sizes, fp32, against the oracle."""
    from paper_2410_23745_b200 import codegen as C
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    torch = _torch()
    ops_ = _corpus()[chunk::8]
    checked = 0
    for op in ops_:
        g, red = reduced_case(op)
        if red is None:
            continue
        h = P.handle_for(g, red, True)
        text = C.emit_loop_nest(g, red)
        rng = np.random.default_rng(1000 + checked)
        xr = _rounded(rng.standard_normal(h.x_shape), "float32")
        wr = [_rounded(rng.standard_normal(s), "float32") for s in h.w_shapes]
        upr = _rounded(rng.standard_normal(h.y_shape), "float32")
        xd, ud = ops.to_device(xr, "float32"), ops.to_device(upr, "float32")
        wd = [ops.to_device(w, "float32") for w in wr]
        gy = ops.forward(h, xd, wd)
        gdx, gdw = ops.backward(h, xd, wd, ud)
        torch.cuda.synchronize()
        bs = h.x_shape[:1]
        f = lambda t: t.double().cpu().numpy()  # noqa: E731
        assert O.rel_err(f(gy), O.interpret(text, red, xr, wr, bs)) < 1e-4, op
        assert O.rel_err(f(gdx), O.input_gradient(text, red, xr, upr, wr, bs)) < 1e-4, op
        for a, b in zip(gdw, O.weight_gradient(text, red, xr, upr, wr, bs) if wr else []):
            assert O.rel_err(f(a), b) < 1e-4, op
        checked += 1
    assert checked >= len(ops_) // 2


@pytest.mark.parametrize("name", ["conv2d_8", "strided_conv1d", "sep_shared", "bpool", "corpus0003", "corpus0011"])
def test_program_fallback_fp32(cuda, name, monkeypatch):
    """The on-the-fly coordinate-program path (what a 2^28-entry table falls
    back to at full size) in float32, tolerance 1e-4."""
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    torch = _torch()
    case = next(c for c in CASES if c["name"] == name)
    monkeypatch.setenv("SYNO_TABLE_LIMIT", "2")
    h = P.Handle(case["document"], case["assignment"], False)
    x, ws, up, _, _, _ = case_tensors(case)
    env, bs = case["env"], case["batch_shape"]
    x, up = _rounded(x, "float32"), _rounded(up, "float32")
    ws = [_rounded(w, "float32") for w in ws]
    xd, ud = ops.to_device(x, "float32"), ops.to_device(up, "float32")
    wd = [ops.to_device(w, "float32") for w in ws]
    gy = ops.forward(h, xd, wd)
    gdx, gdw = ops.backward(h, xd, wd, ud)
    torch.cuda.synchronize()
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    assert O.rel_err(f(gy), O.interpret(case["nest"], env, x, ws, bs)) < 1e-4
    assert O.rel_err(f(gdx), O.input_gradient(case["nest"], env, x, up, ws, bs)) < 1e-4
    for a, b in zip(gdw, O.weight_gradient(case["nest"], env, x, up, ws, bs) if ws else []):
        assert O.rel_err(f(a), b) < 1e-4


@pytest.mark.parametrize("chunk", range(4))
def test_corpus_program_fallback_reduced_fp32(cuda, chunk, monkeypatch):
    """Corpus operators with every index table forced onto the program path
    (SYNO_TABLE_LIMIT=2), fp32 at reduced sizes, against the oracle."""
    from paper_2410_23745_b200 import codegen as C
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    torch = _torch()
    monkeypatch.setenv("SYNO_TABLE_LIMIT", "2")
    checked = 0
    for op in _corpus()[chunk::16]:
        g, red = reduced_case(op)
        if red is None:
            continue
        for staged in (False, True):
            h = P.Handle(P.operator_document(g), red, staged)
            text = C.emit_loop_nest(g, red)
            rng = np.random.default_rng(2000 + checked)
            xr = _rounded(rng.standard_normal(h.x_shape), "float32")
            wr = [_rounded(rng.standard_normal(s), "float32") for s in h.w_shapes]
            upr = _rounded(rng.standard_normal(h.y_shape), "float32")
            xd, ud = ops.to_device(xr, "float32"), ops.to_device(upr, "float32")
            wd = [ops.to_device(w, "float32") for w in wr]
            gy = ops.forward(h, xd, wd)
            gdx, gdw = ops.backward(h, xd, wd, ud)
            torch.cuda.synchronize()
            bs = h.x_shape[:1]
            f = lambda t: t.double().cpu().numpy()  # noqa: E731
            assert O.rel_err(f(gy), O.interpret(text, red, xr, wr, bs)) < 1e-4, op
            assert O.rel_err(f(gdx), O.input_gradient(text, red, xr, upr, wr, bs)) < 1e-4, op
            for a, b in zip(gdw, O.weight_gradient(text, red, xr, upr, wr, bs) if wr else []):
                assert O.rel_err(f(a), b) < 1e-4, op
        checked += 1
    assert checked >= 10


def _full_size_spot_ids(count=16, max_grid=1 << 24):
    """Seeded choice of corpus candidates whose full-size (one image) grid the
    oracle evaluates in seconds: half with weights, half pure gathers."""
    from paper_2410_23745_b200 import codegen as C
    from paper_2410_23745_b200 import pgraph as P
    spec = P.build_spec(**dict(CORPUS_SPEC, reference=dict(CORPUS_SPEC["reference"], N=1)))
    rng = np.random.default_rng(8)
    weighted, plain = [], []
    for i in rng.permutation(len(_corpus())):
        g = P.parse_steps(_corpus()[i], spec)
        try:
            if C.flops(g) // 2 > max_grid:
                continue
        except Exception:
            continue
        bucket = weighted if g.n_weights else plain
        if len(bucket) < count // 2:
            bucket.append(int(i))
        if len(weighted) + len(plain) == count:
            break
    return sorted(weighted + plain)


@pytest.mark.parametrize("staged", [False, True], ids=["unstaged", "staged"])
def test_corpus_full_size_oracle_spot_check(cuda, staged):
    """a seeded subset of corpus candidates at FULL size
    (C=64, H=W=32, one image), fp32, forward + grad-input + grad-weight
    against the oracle (reference codegen.py:598-743)."""
    from paper_2410_23745_b200 import codegen as C
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    torch = _torch()
    spec = P.build_spec(**dict(CORPUS_SPEC, reference=dict(CORPUS_SPEC["reference"], N=1)))
    ids = _full_size_spot_ids()
    assert len(ids) == 16
    for i in ids:
        g = P.parse_steps(_corpus()[i], spec)
        h = P.handle_for(g, None, staged)
        env = dict(CORPUS_SPEC["reference"], N=1)
        text = C.emit_loop_nest(g)
        rng = np.random.default_rng(3000 + i)
        xr = _rounded(rng.standard_normal(h.x_shape), "float32")
        wr = [_rounded(rng.standard_normal(s), "float32") for s in h.w_shapes]
        upr = _rounded(rng.standard_normal(h.y_shape), "float32")
        xd, ud = ops.to_device(xr, "float32"), ops.to_device(upr, "float32")
        wd = [ops.to_device(w, "float32") for w in wr]
        gy = ops.forward(h, xd, wd)
        gdx, gdw = ops.backward(h, xd, wd, ud)
        torch.cuda.synchronize()
        f = lambda t: t.double().cpu().numpy()  # noqa: E731
        assert O.rel_err(f(gy), O.interpret(text, env, xr, wr, (1,))) < 1e-4, i
        assert O.rel_err(f(gdx), O.input_gradient(text, env, xr, upr, wr, (1,))) < 1e-4, i
        for a, b in zip(gdw, O.weight_gradient(text, env, xr, upr, wr, (1,)) if wr else []):
            assert O.rel_err(f(a), b) < 1e-4, i


# the heaviest sweep candidates (program fallback / 2^28-entry tables at
# N=8), sample 828 among them
HEAVY = [828, 170, 171, 172, 732, 736, 518, 7, 8, 319]


@pytest.mark.parametrize("sid", HEAVY)
def test_heavy_sweep_candidates_adjoint_f64(cuda, sid):
    """Full sweep size (N=8): the float64 run must satisfy the adjoint
    identities <dy, y> = <dx, x> = <dw_j, w_j> to 1e-10 (what the sweep
    checks in fp32 to 1e-4), and the fp32 run must agree with the f64 run
    to 1e-4 in y, dx and every dw."""
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import workloads as WL
    from paper_2410_23745_b200.sweep import evaluate
    torch = _torch()
    g = WL.corpus(8)[sid]
    r = evaluate(g, sid, sid, dtype=torch.float64)
    assert r.status == "ok" and r.adjoint_err < 1e-10, r
    r32 = evaluate(g, sid, sid, dtype=torch.float32)
    assert r32.status == "ok", r32
    from paper_2410_23745_b200 import pgraph as P
    h = P.handle_for(g, None, True)
    gen = torch.Generator(device="cuda").manual_seed(sid)
    x = torch.randn(h.x_shape, generator=gen, device="cuda", dtype=torch.float64)
    ws = [torch.randn(s, generator=gen, device="cuda", dtype=torch.float64) for s in h.w_shapes]
    dy = torch.randn(h.y_shape, generator=gen, device="cuda", dtype=torch.float64)
    x, ws, dy = x.float().double(), [w.float().double() for w in ws], dy.float().double()
    y64 = ops.forward(h, x, ws)
    dx64, dw64 = ops.backward(h, x, ws, dy)
    y32 = ops.forward(h, x.float(), [w.float() for w in ws])
    dx32, dw32 = ops.backward(h, x.float(), [w.float() for w in ws], dy.float())
    torch.cuda.synchronize()
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    assert O.rel_err(f(y32), f(y64)) < 1e-4
    assert O.rel_err(f(dx32), f(dx64)) < 1e-4
    for a, b in zip(dw32, dw64):
        assert O.rel_err(f(a), f(b)) < 1e-4


# weighted corpus candidates of the gathered-GEMM form
# y[b, n, m] = sum_r x[gx(b, m, r)] * w[gw(n, r)] (engine.cu GatherGemm)
GATHERED_GEMM = [171, 1016, 792, 179, 197, 319, 381, 688]


@pytest.mark.parametrize("sid", GATHERED_GEMM)
@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_gathered_gemm_candidates(cuda, sid, dtype):
    """Sampled contractions with gathered operands run on the tcgen05 path
    (the profile shows tensor-core GEMM launches) and match the float64
    universal engine (itself pinned to the oracle) on the same inputs:
    fp32 1e-4, bf16 2e-2 (inputs rounded to the dtype first)."""
    from paper_2410_23745_b200 import _lib, ops
    from paper_2410_23745_b200 import pgraph as P
    from paper_2410_23745_b200 import workloads as WL
    torch = _torch()
    g = WL.corpus(2)[sid]
    h = P.handle_for(g, None, True)
    dt = getattr(torch, dtype)
    gen = torch.Generator(device="cuda").manual_seed(sid)
    x = torch.randn(h.x_shape, generator=gen, device="cuda").to(dt)
    ws = [torch.randn(s, generator=gen, device="cuda").to(dt) for s in h.w_shapes]
    dy = torch.randn(h.y_shape, generator=gen, device="cuda").to(dt)
    _lib.profile_begin()
    y = ops.forward(h, x, ws)
    dx, dws = ops.backward(h, x, ws, dy)
    torch.cuda.synchronize()
    prof = _lib.profile_end()
    if sid != 688:
        assert any(k.startswith("tc_gemm") for k in prof), (sid, sorted(prof))
    y64 = ops.forward(h, x.double(), [w.double() for w in ws])
    dx64, dw64 = ops.backward(h, x.double(), [w.double() for w in ws], dy.double())
    tol = TOL[dtype]
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    assert O.rel_err(f(y), f(y64)) < tol
    assert O.rel_err(f(dx), f(dx64)) < tol
    for a, b in zip(dws, dw64):
        assert O.rel_err(f(a), f(b)) < tol

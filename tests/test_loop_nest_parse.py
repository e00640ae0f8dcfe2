"""Native parse_loop_nest (csrc/nest.cpp, codegen.py:846-943) and run_nest.

The emitted nest text is byte-identical to the reference's
(test_lowering.py), so `emit(parse(text)) == text` on the reference's own
golden text is the reference's round-trip test
(pkg/tests/test_codegen.py:428-435) on its own fixtures.  Execution of a
parsed nest (pkg/tests/test_codegen.py:438-444) is in the GPU half below.
"""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from conftest import CASE_IDS, CASES, GOLDEN, case_tensors

from paper_2410_23745_b200 import codegen as C
from paper_2410_23745_b200 import pgraph as P
from paper_2410_23745_b200.errors import LoopNestParseError, ShapeMismatch, UnsupportedOperator

CONV_SPEC = ("conv2d", ("C_out", "C_in", "H", "W"), ("K",), {"C_out": 8, "C_in": 8, "H": 8, "W": 8, "K": 3},
             ("C_out", "H", "W"), ("C_in", "H", "W"))


def _spec_of(case):
    return P.parse_operator(case["document"]).spec


@pytest.mark.parametrize("case", CASES, ids=CASE_IDS)
def test_golden_nest_text_round_trips(case):
    spec = _spec_of(case)
    env = case["env"]
    for key in ("nest", "nest_staged"):
        n = C.parse_loop_nest(case[key], spec, env)
        assert C.emit_loop_nest(n) == case[key]
        assert n == C.parse_loop_nest(case[key], spec, env)
    staged = C.parse_loop_nest(case["nest_staged"], spec, env)
    assert staged.n_stages == case["n_stages"]


def test_corpus_nests_round_trip():
    spec = P.build_spec("conv64", ("C_out", "C_in", "H", "W", "N"), ("K", "s"),
                        {"C_out": 64, "C_in": 64, "H": 32, "W": 32, "K": 3, "s": 2, "N": 8},
                        ("C_out", "H", "W"), ("C_in", "H", "W"), ("N",))
    ops = [ln.strip() for ln in open(os.path.join(GOLDEN, "corpus_conv64.txt")) if ln.strip()]
    for op in ops[::4]:
        g = P.parse_steps(op, spec)
        for staged in (False, True):
            text = C.emit_loop_nest(g, staged=staged)
            n = C.parse_loop_nest(text, spec)
            assert C.emit_loop_nest(n) == text, op
            h = P.handle_for(g)
            assert n.handle.w_shapes == h.w_shapes
            assert tuple(n.handle.x_shape) == tuple(h.x_shape[1:])  # run_nest has no batch axis


def test_spaces_and_blank_lines_are_tolerated():
    spec = P.build_spec(*CONV_SPEC)
    g = P.parse_steps("op{reduce(C_in); contract[0:weight,3:both]}", P.build_spec(
        "pw", ("C_out", "C_in", "H", "W"), (), {"C_out": 8, "C_in": 8, "H": 8, "W": 8}, ("C_out", "H", "W"),
        ("C_in", "H", "W")))
    text = C.emit_loop_nest(g)
    messy = "\n\n" + text.replace("\n", "\n\n") + "   \n"
    assert C.emit_loop_nest(C.parse_loop_nest(messy, g.spec)) == text
    del spec


@pytest.mark.parametrize("bad", [
    "",
    "tensor x = input[C_in]\n",
    "nest n\ntensor x = bogus[C_in]\n",
    "nest n\ntensor x = input[C_in, H, W]\nfor i in C_out:\n  y[i] = x[q]\n",
    "nest n\ntensor x = input[C_in, H, W]\nfor i in C_out:\n  acc = 0\n  for r in C_in:\n    acc = x[r]\n",
    "nest n\ntensor x = input[C_in, H, W]\nfor i in C_out:\n  acc = 0\n  for r in C_in:\n    acc += x[r]\n  y = x\n",
    "nest n\ntensor x = input[C_in, H, W]\nfor i in C_out:\n  y[i] = x[(i]\n",
    "nest n\ntensor x = input[C_in, H, W]\nfor i in C_out:\n  y[i] = x[i $ 2]\n",
    "nest n\ntensor x = input[C_in, H, W]\nfor i in C_out:\n  y[i] = 3 + \n",
    "nest n\ntensor x = input[C_in, H, W]\ntensor y = output[C_out, H, W]\nfor i in C_out:\n  y[i] = x[i] * 2\n",
])
def test_malformed_text_raises_loop_nest_parse_error(bad):
    with pytest.raises(LoopNestParseError):
        C.parse_loop_nest(bad, P.build_spec(*CONV_SPEC))


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree absent (GPU box)")
def test_reference_parser_agrees_on_edge_texts():
    """The reference's parse_loop_nest accepts / rejects the same texts, and
    what it accepts re-emits to the same bytes here."""
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from opsmith import codegen as RC
    from opsmith.pgraph import ProblemSpec
    from opsmith.symexpr import Variable, parse_size

    name, prim, coeffs, ref, out, inp = CONV_SPEC
    vs = tuple(Variable(n) for n in prim) + tuple(Variable(n, primary=False) for n in coeffs)
    vm = {v.name: v for v in vs}
    rspec = ProblemSpec(name=name, variables=vs, reference=tuple(ref.items()),
                        output_dims=tuple(parse_size(t, vm) for t in out),
                        input_dims=tuple(parse_size(t, vm) for t in inp))
    texts = [
        "nest n\ntensor x = input[C_in, H, W]\ntensor y = output[C_out, H, W]\n"
        "for a in C_out:\n  for b in H:\n    for c in W:\n      y[a, b, c] = x[a % C_in, (b + 1) % H, c * 1]\n",
        "nest n\ntensor x = input[C_in, H, W]\ntensor t0 = stage[8, 8]\ntensor y = output[C_out, H, W]\n"
        "for a in 8:\n  for b in 8:\n    acc = 0\n    for r in C_in:\n      acc += x[r, a, b]\n    t0[a, b] = acc\n"
        "for a in C_out:\n  for b in H:\n    for c in W:\n      y[a, b, c] = t0[b, c]\n",
        "nest n\ntensor x = input[C_in, H, W]\ntensor y = output[C_out, H, W]\n"
        "for a in C_out:\n  for b in H:\n    for c in W:\n      y[a, b, c] = x[a / K^2, b - K*C_in + K*C_in, c]\n",
    ]
    for t in texts:
        want = RC.emit_loop_nest(RC.parse_loop_nest(t, rspec))
        assert C.emit_loop_nest(C.parse_loop_nest(t, P.build_spec(*CONV_SPEC))) == want
    for bad in ("nest n\nfor i in C_out:\n  y[i] = x[(i]\n", "nest n\ntensor x = bogus[C_in]\n"):
        with pytest.raises(ValueError):
            RC.parse_loop_nest(bad, rspec)
        with pytest.raises(ValueError):
            C.parse_loop_nest(bad, P.build_spec(*CONV_SPEC))


# ---------------------------------------------------------------------------
# GPU: run_nest on parsed nests (pkg/tests/test_codegen.py:438-444)
# ---------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=CASE_IDS)
def test_run_parsed_nest_matches_reference_values(case):
    import torch
    assert torch.cuda.is_available()
    spec = _spec_of(case)
    env = case["env"]
    x, ws, up, y, y_staged, dws = case_tensors(case)
    nb = len(case["batch_shape"])
    xe = x.reshape((-1,) + x.shape[nb:])[0]
    for key, want in (("nest", y), ("nest_staged", y_staged)):
        n = C.parse_loop_nest(case[key], spec, env)
        got = C.run_nest(n, xe, ws)
        ref = want.reshape((-1,) + want.shape[nb:])[0]
        assert np.abs(got - ref).max() <= 1e-10 * max(np.abs(ref).max(), 1e-12), (case["name"], key)


@pytest.mark.gpu
def test_parsed_single_stage_nest_has_a_backward():
    import torch
    from paper_2410_23745_b200 import ops
    spec = P.build_spec(*CONV_SPEC)
    g = P.parse_steps("op{reduce(C_in); reduce(K); reduce(K); contract[0:weight,3:both,4:both,5:both]; "
                      "unfold[1,7]; unfold[2,8]}", spec)
    n = C.parse_loop_nest(C.emit_loop_nest(g), spec)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(n.handle.x_shape)
    (w,) = [rng.standard_normal(s) for s in n.handle.w_shapes]
    up = rng.standard_normal(n.handle.y_shape)
    dx, (dw,) = ops.backward(n.handle, ops.to_device(x, "float64"), [ops.to_device(w, "float64")],
                             ops.to_device(up, "float64"))
    gdx, (gdw,) = C.gradients(g, x, up, [w])  # the spec has no batch dims: same shapes
    assert np.abs(ops.to_numpy(dx) - gdx).max() < 1e-10 * np.abs(gdx).max()
    assert np.abs(ops.to_numpy(dw) - gdw).max() < 1e-10 * np.abs(gdw).max()
    with pytest.raises(ShapeMismatch):
        C.run_nest(n, x[None], [w])
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_parsed_staged_nest_is_forward_only():
    from paper_2410_23745_b200 import ops
    spec = P.build_spec("conv64", ("C_out", "C_in", "H", "W"), ("K",),
                        {"C_out": 8, "C_in": 8, "H": 8, "W": 8, "K": 3}, ("C_out", "H", "W"), ("C_in", "H", "W"))
    g = P.parse_steps("op{reduce(C_in); reduce(K); reduce(K); contract[0:weight,3:both,4:both]; "
                      "unfold[1,7]; contract[5:both]; unfold[2,9]}", spec)
    n = C.parse_loop_nest(C.emit_loop_nest(g, staged=True), spec)
    assert n.n_stages > 1
    rng = np.random.default_rng(4)
    x = rng.standard_normal(n.handle.x_shape)
    ws = [rng.standard_normal(s) for s in n.handle.w_shapes]
    want = C.interpret(g, x, ws, staged=True)
    got = C.run_nest(n, x, ws)
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    with pytest.raises(UnsupportedOperator):
        ops.backward(n.handle, ops.to_device(x, "float64"), [ops.to_device(w, "float64") for w in ws],
                     ops.to_device(rng.standard_normal(n.handle.y_shape), "float64"))

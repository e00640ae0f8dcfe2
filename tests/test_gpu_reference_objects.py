"""GPU: the reference's own PGraph objects through the patched API.

INTEGRATION.md's opt-in rebinding makes ``opsmith.codegen.interpret`` and
``weight_gradient`` the backend's; the reference's callers then pass their
own graphs and numpy arrays and get float64 numpy results computed on the
B200.  The reference package comes from baseline/_ref (the pip --target
install that travels to the GPU box) or the source tree in the build
container; the test is skipped when neither exists.  Results are compared
with the reference's unpatched functions on the same inputs (float64,
1e-10, reference test_codegen.py:95-97).
"""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _opsmith():
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "opsmith")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import opsmith.codegen as RC
            import opsmith.pgraph as RP
            import opsmith.symexpr as RS
            return RC, RP, RS
    pytest.skip("reference package not installed (baseline/_ref)")


def _graph(RP, RS, spec_args, steps):
    name, prim, coeffs, refv, out, inp, batch = spec_args
    variables = tuple(RS.Variable(n) for n in prim) + tuple(RS.Variable(n, primary=False) for n in coeffs)
    vm = {v.name: v for v in variables}
    spec = RP.ProblemSpec(name=name, variables=variables, reference=tuple(refv.items()),
                          output_dims=tuple(RS.parse_size(t, vm) for t in out),
                          input_dims=tuple(RS.parse_size(t, vm) for t in inp),
                          batch_dims=tuple(RS.parse_size(t, vm) for t in batch))
    return RP.parse_steps(steps, spec)


def test_patched_interpret_and_weight_gradient_on_reference_graphs(cuda, monkeypatch):
    RC, RP, RS = _opsmith()
    from paper_2410_23745_b200 import codegen as B
    from paper_2410_23745_b200 import configs as CF
    small = {"C_out": 8, "C_in": 4, "H": 6, "W": 5, "K": 3, "s": 2, "N": 2}
    cases = [_graph(RP, RS, CF.conv_spec_args("c", op, 4, 8, 6, 2), CF.STEPS[op])
             for op in ("conv3x3", "sep_shared", "conv3x3_s2", "pointwise")]
    spec = CF.corpus_spec_args(2)
    spec = (spec[0], spec[1], spec[2], dict(small), spec[4], spec[5], spec[6])
    for op in CF.corpus_ops()[:200:10]:
        try:
            g = _graph(RP, RS, spec, op)
            RC.build_loop_nest(g)
        except Exception:
            continue
        cases.append(g)
    assert len(cases) >= 10
    orig_i, orig_w = RC.interpret, RC.weight_gradient
    monkeypatch.setattr(RC, "interpret", B.interpret)
    monkeypatch.setattr(RC, "weight_gradient", B.weight_gradient)
    rng = np.random.default_rng(0)
    for g in cases:
        x = rng.standard_normal(RC.input_shape(g.spec))
        ws = RC.random_weights(g, rng)
        up = rng.standard_normal(RC.output_shape(g.spec))
        y = RC.interpret(g, x, ws)
        want = orig_i(g, x, ws)
        assert isinstance(y, np.ndarray) and y.dtype == np.float64
        assert float(np.abs(y - want).max()) <= 1e-10 * max(1.0, float(np.abs(want).max())), RP.print_steps(g)
        if ws:
            for a, b in zip(RC.weight_gradient(g, x, up, ws), orig_w(g, x, up, ws)):
                assert float(np.abs(a - b).max()) <= 1e-10 * max(1.0, float(np.abs(b).max())), RP.print_steps(g)

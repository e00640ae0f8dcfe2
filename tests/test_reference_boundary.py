"""The drop-in boundary on the REFERENCE's own objects (CPU).

INTEGRATION.md's opt-in patch rebinds ``opsmith.codegen.flops`` /
``param_count`` / ``interpret`` / ``weight_gradient`` to this package's
functions, which then receive the reference's own ``PGraph`` objects
(duck-typed through ``pgraph.operator_document``, pgraph.py:108-125).  Here
the patch is applied to the real reference package (imported from
/root/reference/pkg/src in this container; skipped where it is absent, e.g.
on the GPU box) and the host-side results are compared with the
reference's unpatched functions across the whole cfg5 corpus and the
config operator set: flops (unstaged and rfactor-staged, codegen.py:633),
param_count (codegen.py:654), the emitted loop nest (codegen.py:750) and
the operator document (pgraph.py:712).  No device is needed for these.
"""
from __future__ import annotations

import os
import sys

import pytest

REF_SRC = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF_SRC, "opsmith")),
                                reason="reference source tree not present")


@pytest.fixture(scope="module")
def ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import opsmith.codegen as RC
    import opsmith.pgraph as RP
    import opsmith.symexpr as RS
    return RC, RP, RS


def _ref_graph(ref, spec_args, steps):
    RC, RP, RS = ref
    name, prim, coeffs, refv, out, inp, batch = spec_args
    variables = tuple(RS.Variable(n) for n in prim) + tuple(RS.Variable(n, primary=False) for n in coeffs)
    vm = {v.name: v for v in variables}
    spec = RP.ProblemSpec(name=name, variables=variables, reference=tuple(refv.items()),
                          output_dims=tuple(RS.parse_size(t, vm) for t in out),
                          input_dims=tuple(RS.parse_size(t, vm) for t in inp),
                          batch_dims=tuple(RS.parse_size(t, vm) for t in batch))
    return RP.parse_steps(steps, spec)


def _graphs(ref):
    from paper_2410_23745_b200 import configs as CF
    out = [_ref_graph(ref, CF.corpus_spec_args(8), op) for op in CF.corpus_ops()]
    for name, op, ci, co, h in CF.resnet18_table() + CF.resnet34_table():
        out.append(_ref_graph(ref, CF.conv_spec_args(name, op, ci, co, h, 4), CF.STEPS[op]))
    out.append(_ref_graph(ref, CF.qkv_spec_args(2, 64), CF.QKV))
    return out


def test_patched_reference_host_queries_match(ref, monkeypatch):
    RC, RP, _ = ref
    from paper_2410_23745_b200 import codegen as B
    orig = {k: getattr(RC, k) for k in ("flops", "param_count", "interpret", "weight_gradient")}
    # the opt-in rebinding inside opsmith.codegen
    for k in orig:
        monkeypatch.setattr(RC, k, getattr(B, k))
    graphs = _graphs(ref)
    assert len(graphs) >= 1024
    for g in graphs:
        assert RC.flops(g) == orig["flops"](g), RP.print_steps(g)
        assert RC.flops(g, staged=True) == orig["flops"](g, staged=True), RP.print_steps(g)
        assert RC.param_count(g) == orig["param_count"](g), RP.print_steps(g)


def test_reference_graphs_emit_identical_nests(ref):
    RC, RP, _ = ref
    from paper_2410_23745_b200 import codegen as B
    from paper_2410_23745_b200 import pgraph as P
    for g in _graphs(ref):
        nest = RC.build_loop_nest(g)
        assert B.emit_loop_nest(g) == RC.emit_loop_nest(nest), RP.print_steps(g)
        assert B.emit_loop_nest(g, staged=True) == RC.emit_loop_nest(RC.rfactor(nest)), RP.print_steps(g)
        # the operator document the boundary builds from a reference PGraph
        # is the reference's own print_operator text
        assert P.operator_document(g) == RP.print_operator(g), RP.print_steps(g)


def test_reference_graph_shapes(ref):
    RC, RP, _ = ref
    from paper_2410_23745_b200 import codegen as B
    for g in _graphs(ref)[::7]:
        assert B.input_shape(g.spec) == RC.input_shape(g.spec)
        assert B.output_shape(g.spec) == RC.output_shape(g.spec)
        assert B.weight_shapes(g) == RC.weight_shapes(g)

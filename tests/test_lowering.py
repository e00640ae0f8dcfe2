"""Native lowering vs the reference's own output (golden fixtures).

Pins: emitted loop-nest text byte-equal to codegen.emit_loop_nest for the
direct nest and the rfactor staging (codegen.py:297-508, 750-794), flops /
param_count (codegen.py:633-657), the operator document round trip
(pgraph.py:712-790) and the reference's error behaviour.
"""
from __future__ import annotations

import pytest

from conftest import CASE_IDS, CASES

from paper_2410_23745_b200 import codegen as C
from paper_2410_23745_b200 import pgraph as P
from paper_2410_23745_b200.errors import OperatorParseError, ShapeMismatch


@pytest.mark.parametrize("case", CASES, ids=CASE_IDS)
def test_emitted_nest_is_byte_identical(case):
    g = P.parse_operator(case["document"])
    env = case["env"]
    assert C.emit_loop_nest(g, env) == case["nest"]
    assert C.emit_loop_nest(g, env, staged=True) == case["nest_staged"]


@pytest.mark.parametrize("case", CASES, ids=CASE_IDS)
def test_flops_and_params(case):
    g = P.parse_operator(case["document"])
    env = case["env"]
    assert C.flops(g, env) == case["flops"]
    assert C.flops(g, env, staged=True) == case["flops_staged"]
    assert C.param_count(g, env) == case["params"]


@pytest.mark.parametrize("case", CASES, ids=CASE_IDS)
def test_document_round_trip(case):
    g = P.parse_operator(case["document"])
    assert P.print_operator(g) == case["document"]
    assert P.print_steps(g) == case["steps"] or case["steps"] == "op{}"


def test_corpus_replays_and_lowers():
    """All 1024 sampled corpus operators replay and lower natively."""
    import os
    from conftest import GOLDEN
    spec = P.build_spec("conv64", ("C_out", "C_in", "H", "W", "N"), ("K", "s"),
                        {"C_out": 64, "C_in": 64, "H": 32, "W": 32, "K": 3, "s": 2, "N": 8},
                        ("C_out", "H", "W"), ("C_in", "H", "W"), ("N",))
    ops = [ln.strip() for ln in open(os.path.join(GOLDEN, "corpus_conv64.txt")) if ln.strip()]
    assert len(ops) == 1024
    for op in ops:
        g = P.parse_steps(op, spec)
        assert g.complete
        assert C.flops(g, staged=True) <= C.flops(g)


def test_parse_errors_follow_the_reference():
    spec = P.build_spec("conv2d", ("C_out", "C_in", "H", "W"), ("K",),
                        {"C_out": 8, "C_in": 8, "H": 8, "W": 8, "K": 3}, ("C_out", "H", "W"), ("C_in", "H", "W"))
    with pytest.raises(OperatorParseError):
        P.parse_steps("reduce(K)", spec)                  # missing op{...}
    with pytest.raises(OperatorParseError):
        P.parse_steps("op{reduce(K); unfold[1,9]}", spec)  # unknown dim
    with pytest.raises(OperatorParseError):
        P.parse_steps("op{unfold[1,2]; reduce(K)}", spec)  # reduce after the stage ended
    with pytest.raises(OperatorParseError):
        P.parse_steps("op{contract[0:sideways]}", spec)
    with pytest.raises(ValueError):
        P.parse_steps("op{reduce(Q)}", spec)              # unknown size variable
    g = P.parse_steps("op{reduce(K)}", spec)              # replays, but incomplete
    assert not g.complete
    with pytest.raises(ShapeMismatch):
        C.flops(g)
    doc = P.parse_steps("op{reduce(C_in); reduce(K); reduce(K); contract[0:weight,3:both,4:both,5:both]; "
                        "unfold[1,7]; unfold[2,8]}", spec).document
    with pytest.raises(OperatorParseError):
        P.parse_operator(doc.replace("perm 0 1 2", "perm 2 1 0"))
    with pytest.raises(OperatorParseError):
        P.parse_operator(doc.replace("var K coefficient 3", "var K scalar 3"))


_SIMPLIFY_CHECK = r"""
import sys
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + '/tests')
from conftest import CASES
from paper_2410_23745_b200 import pgraph as P
from paper_2410_23745_b200 import workloads as WL
n = 0
for staged in (False, True):
    for g in WL.corpus(8) + WL.corpus(1):
        P.Handle(P.operator_document(g), None, staged)
        n += 1
    for c in CASES:
        P.Handle(c["document"], c["assignment"], staged)
        n += 1
print("checked", n)
"""


def test_coordinate_simplification_is_exact():
    """The engine's quasi-affine rewrite of every coordinate (csrc/simplify.cpp)
    leaves each value unchanged: SYNO_CHECK_SIMPLIFY compares rewritten and
    original expressions at the loop-range corners and 4096 pseudo-random
    grid points, for every stage (forward, staged forward, grad-input,
    grad-weight, staged backward) of the whole corpus and the golden cases."""
    import os
    import subprocess
    import sys

    from conftest import ROOT
    env = dict(os.environ, SYNO_CHECK_SIMPLIFY="1")
    r = subprocess.run([sys.executable, "-c", _SIMPLIFY_CHECK, ROOT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "checked" in r.stdout

"""Pin the CPU oracle (oracle/nest_oracle.py) to the reference's own outputs.

Every golden case was produced by the reference package itself
(tests/golden/make_golden.py): interpret (codegen.py:598), interpret with
staged=True (rfactor, codegen.py:490) and weight_gradient (codegen.py:664).
grad-input has no reference function; it is pinned by the adjoint identity
<up, A x> = <dX, x> and by central differences in x.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import CASE_IDS, CASES, case_tensors

from oracle import nest_oracle as O


@pytest.mark.parametrize("case", CASES, ids=CASE_IDS)
def test_oracle_interpret_matches_reference(case):
    x, ws, up, y, ys, dws = case_tensors(case)
    env, bs = case["env"], case["batch_shape"]
    got = O.interpret(case["nest"], env, x, ws, bs)
    assert got.shape == y.shape
    assert O.rel_err(got, y) < 1e-12
    got_s = O.interpret(case["nest_staged"], env, x, ws, bs)
    assert O.rel_err(got_s, ys) < 1e-12


@pytest.mark.parametrize("case", [c for c in CASES if c["n_weights"]], ids=[c["name"] for c in CASES if c["n_weights"]])
def test_oracle_weight_gradient_matches_reference(case):
    x, ws, up, y, ys, dws = case_tensors(case)
    got = O.weight_gradient(case["nest"], case["env"], x, up, ws, case["batch_shape"])
    for g, want in zip(got, dws):
        assert O.rel_err(g, want) < 1e-12


@pytest.mark.parametrize("case", CASES, ids=CASE_IDS)
def test_oracle_input_gradient_is_the_adjoint(case):
    x, ws, up, y, ys, dws = case_tensors(case)
    env, bs = case["env"], case["batch_shape"]
    dx = O.input_gradient(case["nest"], env, x, up, ws, bs)
    assert dx.shape == x.shape
    lhs = float(np.sum(up * y))
    rhs = float(np.sum(dx * x))
    assert abs(lhs - rhs) <= 1e-9 * max(1.0, abs(lhs))


@pytest.mark.parametrize("name", ["conv2d_8", "strided_conv1d", "sep_shared", "smooth1d", "corpus0003"])
def test_oracle_input_gradient_central_differences(name):
    case = next(c for c in CASES if c["name"] == name)
    x, ws, up, *_ = case_tensors(case)
    env, bs = case["env"], case["batch_shape"]
    dx = O.input_gradient(case["nest"], env, x, up, ws, bs)
    rng = np.random.default_rng(5)
    for flat in rng.choice(x.size, size=min(6, x.size), replace=False):
        idx = np.unravel_index(flat, x.shape)
        h = 1e-4
        xp, xm = x.copy(), x.copy()
        xp[idx] += h
        xm[idx] -= h
        fp = float(np.sum(up * O.interpret(case["nest"], env, xp, ws, bs)))
        fm = float(np.sum(up * O.interpret(case["nest"], env, xm, ws, bs)))
        fd = (fp - fm) / (2 * h)
        assert abs(dx[idx] - fd) <= 1e-6 * max(1.0, abs(fd))


def test_floor_semantics_pin():
    # test_symexpr.py:93-114: (C*i+j)%(B*C) == 4; floor div/mod of negatives
    e = O.parse_expr("(C * i + j) % (B*C)", {"i", "j"})
    assert int(O.eval_grid(e, {"i": np.int64(5), "j": np.int64(1)}, {"B": 4, "C": 3})) == 4
    e = O.parse_expr("(i - K) / K", {"i"})
    assert int(O.eval_grid(e, {"i": np.int64(1)}, {"K": 3})) == -1
    e = O.parse_expr("(i - K) % K", {"i"})
    assert int(O.eval_grid(e, {"i": np.int64(1)}, {"K": 3})) == 1

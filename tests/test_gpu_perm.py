"""Lane-contiguous permuted layouts (engine.cu lane_contiguous_layout) and
linear-form table compression (engine.cu linear_form).

Heavy gather stages read a copy of their lead input with the unit-stride
dimension innermost, and heavy scatters accumulate into a permuted target
that a restore stage writes back.  The transform only fires above 2^22 grid
points, which the reduced parity cases never reach, so these tests rerun
the reduced corpus (unstaged and staged, every stage) and the golden cases
in a child process with SYNO_PERM_MIN_POINTS=1 (the library reads it once
per process) against the oracle, and check that the transform fired.
"""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import numpy as np, torch
from oracle import nest_oracle as O
from paper_2410_23745_b200 import codegen as C, ops, pgraph as P
import test_gpu_parity as T
ops_ = T._corpus()[{start}::{step}]
checked = 0
for staged in (False, True):
    for op in ops_:
        g, red = T.reduced_case(op)
        if red is None:
            continue
        h = P.handle_for(g, red, staged)
        text = C.emit_loop_nest(g, red)
        rng = np.random.default_rng(7 + checked)
        xr = T._rounded(rng.standard_normal(h.x_shape), "float32")
        wr = [T._rounded(rng.standard_normal(s), "float32") for s in h.w_shapes]
        upr = T._rounded(rng.standard_normal(h.y_shape), "float32")
        xd, ud = ops.to_device(xr, "float32"), ops.to_device(upr, "float32")
        wd = [ops.to_device(w, "float32") for w in wr]
        gy = ops.forward(h, xd, wd)
        gdx, gdw = ops.backward(h, xd, wd, ud)
        torch.cuda.synchronize()
        bs = h.x_shape[:1]
        f = lambda t: t.double().cpu().numpy()
        assert O.rel_err(f(gy), O.interpret(text, red, xr, wr, bs)) < 1e-4, op
        assert O.rel_err(f(gdx), O.input_gradient(text, red, xr, upr, wr, bs)) < 1e-4, op
        for a, b in zip(gdw, O.weight_gradient(text, red, xr, upr, wr, bs) if wr else []):
            assert O.rel_err(f(a), b) < 1e-4, op
        checked += 1
print("checked", checked)
"""


@pytest.mark.gpu
@pytest.mark.parametrize("start", [0, 1])
def test_forced_linear_form_tables_match_oracle(cuda, start):
    """Every mixed table whose coordinate reads its axes through one linear
    form is built over that form (threshold forced to 1)."""
    env = dict(os.environ, SYNO_LINFORM_MIN="1")
    code = CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"), start=start, step=2)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "checked" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("start", [0, 1, 2, 3])
def test_forced_permuted_layouts_match_oracle(cuda, start):
    env = dict(os.environ, SYNO_PERM_MIN_POINTS="1", SYNO_PERM_LOG="1")
    code = CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"), start=start, step=4)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "checked" in r.stdout
    # the transform fired on some stages (gather inputs and scatter targets)
    assert r.stderr.count("[perm] stage gather") > 10 and r.stderr.count("[perm] stage scatter") > 10

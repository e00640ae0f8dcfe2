"""cfg4's sampled QKV variants (tests/golden/corpus_qkv.txt, drawn by the
reference sampler) fwd + bwd on staged handles -- the bench.py
``--workload qkv_variants`` path -- against the oracle at a reduced
assignment, fp32 1e-4 and bf16 2e-2 (reference metric)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import nest_oracle as O
from test_gpu_parity import _rounded

RED = {"T": 32, "E": 24, "E3": 72, "B": 2}


def _ops():
    from paper_2410_23745_b200.configs import qkv_variant_ops
    return qkv_variant_ops()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_qkv_variants_match_oracle(cuda, dtype):
    import torch

    from paper_2410_23745_b200 import codegen as C
    from paper_2410_23745_b200 import ops
    from paper_2410_23745_b200 import pgraph as P
    from paper_2410_23745_b200.configs import qkv_spec_args
    spec = P.build_spec(*qkv_spec_args(16))
    tol = 1e-4 if dtype == "float32" else 2e-2
    checked = 0
    for i, op in enumerate(_ops()):
        g = P.parse_steps(op, spec)
        try:
            h = P.handle_for(g, RED, True)
        except Exception:
            continue  # the reduced assignment does not divide this variant's sizes
        text = C.emit_loop_nest(g, RED)
        rng = np.random.default_rng(50 + i)
        rnd = lambda shape: _rounded(rng.standard_normal(shape), dtype)  # noqa: E731
        x, up = rnd(h.x_shape), rnd(h.y_shape)
        ws = [rnd(s) for s in h.w_shapes]
        xd, ud = ops.to_device(x, dtype), ops.to_device(up, dtype)
        wd = [ops.to_device(w, dtype) for w in ws]
        y = ops.forward(h, xd, wd)
        dx, dws = ops.backward(h, xd, wd, ud)
        torch.cuda.synchronize()
        f = lambda t: t.double().cpu().numpy()  # noqa: E731
        bs = h.x_shape[:1]
        assert O.rel_err(f(y), O.interpret(text, RED, x, ws, bs)) < tol, op
        assert O.rel_err(f(dx), O.input_gradient(text, RED, x, up, ws, bs)) < tol, op
        for a, b in zip(dws, O.weight_gradient(text, RED, x, up, ws, bs)):
            assert O.rel_err(f(a), b) < tol, op
        checked += 1
    assert checked >= 12

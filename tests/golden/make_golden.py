"""Generate golden fixtures FROM THE REFERENCE (this container only).

Imports the read-only reference package from /root/reference/pkg/src and
records, for every case, what the reference itself produces:

  * the operator document          pgraph.print_operator     (pgraph.py:712)
  * the lowered nest text          codegen.emit_loop_nest    (codegen.py:750)
    of build_loop_nest and of rfactor(build_loop_nest)
  * flops (staged/unstaged), param_count                     (codegen.py:633-657)
  * y = interpret(x, w), y_staged = interpret(..., staged=True)
  * dW = weight_gradient(x, up, w)                           (codegen.py:664)

on inputs drawn from np.random.default_rng(seed).standard_normal, the
reference's own random_weights convention (codegen.py:590-595).

Outputs: tests/golden/cases.json and tests/golden/tensors.npz.  The GPU
box never runs this; tests read the committed fixtures.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from opsmith import codegen as C  # noqa: E402
from opsmith.pgraph import ProblemSpec, parse_steps, print_operator  # noqa: E402
from opsmith.symexpr import NonIntegralSize, Variable, parse_size  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CONV_STEPS = ("op{reduce(C_in); reduce(K); reduce(K); "
              "contract[0:weight,3:both,4:both,5:both]; unfold[1,7]; unfold[2,8]}")
CONV_S2 = ("op{reduce(C_in); reduce(K); reduce(K); contract[0:weight,3:both,4:both,5:both]; "
           "stride(s)[1]; unfold[9,7]; stride(s)[2]; unfold[11,8]}")
SEP_SHARED = ("op{reduce(C_in); reduce(K); reduce(K); contract[0:weight,3:both,4:both]; "
              "unfold[1,7]; contract[5:both]; unfold[2,9]}")
POINTWISE = "op{reduce(C_in); contract[0:weight,3:both]}"
SUMPOOL = "op{reduce(K); reduce(K); unfold[1,3]; unfold[2,4]}"
QKV = "op{reduce(E); contract[1:weight,2:both]}"


def spec(name, primaries, coeffs, ref, output, input_, batch=()):
    variables = tuple(Variable(n) for n in primaries) + tuple(Variable(n, primary=False) for n in coeffs)
    vm = {v.name: v for v in variables}
    return ProblemSpec(
        name=name, variables=variables, reference=tuple(ref.items()),
        output_dims=tuple(parse_size(t, vm) for t in output),
        input_dims=tuple(parse_size(t, vm) for t in input_),
        batch_dims=tuple(parse_size(t, vm) for t in batch),
    )


def conv_spec(ref, batch=True, s2=False, same_c=False):
    prims = ("C_out", "C_in", "H", "W") + (("N",) if batch else ())
    inp = ("C_in", "s*H", "s*W") if s2 else ("C_in", "H", "W")
    if same_c:
        return spec("pool", ("C", "H", "W") + (("N",) if batch else ()), ("K",), ref,
                    ("C", "H", "W"), ("C", "H", "W"), ("N",) if batch else ())
    return spec("conv", prims, ("K", "s") if s2 else ("K",), ref, ("C_out", "H", "W"), inp,
                ("N",) if batch else ())


def reference_fixture_cases():
    """The reference's own test operators (tests/conftest.py, tests/test_codegen.py:104-157)."""
    cases = []
    cases.append(("conv2d_8", spec("conv2d", ("C_out", "C_in", "H", "W"), ("K",),
                                   {"C_out": 8, "C_in": 8, "H": 8, "W": 8, "K": 3},
                                   ("C_out", "H", "W"), ("C_in", "H", "W")), CONV_STEPS, None, 7))
    pool = spec("pool1d", ("C", "H"), ("K",), {"C": 4, "H": 16, "K": 5}, ("C", "H"), ("C", "H"))
    cases.append(("pool1d", pool, "op{reduce(K); unfold[1,2]}", None, 8))
    cases.append(("avg_pool1d", pool, "op{reduce(K); contract[2:both]; unfold[1,3]}", None, 8))
    cases.append(("strided_conv1d", spec("strided_conv", ("C_out", "H"), ("C_in", "K", "s"),
                                         {"C_out": 4, "H": 8, "C_in": 3, "K": 3, "s": 2},
                                         ("C_out", "H"), ("C_in", "s*H")),
                  "op{reduce(C_in); reduce(K); contract[0:weight,2:both,3:both]; stride(s)[1]; unfold[6,5]}",
                  None, 9))
    cases.append(("matmul", spec("matmul", ("M", "N"), ("K",), {"M": 6, "N": 7, "K": 5}, ("M", "N"), ("K", "N")),
                  "op{reduce(K); contract[0:weight,2:both]}", None, 10))
    cases.append(("smooth1d", spec("smooth1d", ("H",), ("k", "s"), {"H": 32, "k": 3, "s": 2}, ("H",), ("H",)),
                  "op{reduce(k); reduce(s); contract[1:both]; unfold[0,2]; unfold[4,3]}", None, 18))
    cases.append(("identity", spec("identity", ("N",), (), {"N": 6}, ("N",), ("N",)), "op{}", None, 4))
    cases.append(("bpool", spec("bpool", ("C", "H"), ("K", "N"), {"C": 3, "H": 8, "K": 3, "N": 4},
                                ("C", "H"), ("C", "H"), batch=("N",)),
                  "op{reduce(K); unfold[1,2]}", None, 13))
    cases.append(("edge_taps", spec("edge", ("H",), ("K",), {"H": 4, "K": 9}, ("H",), ("H",)),
                  "op{reduce(K); contract[1:both]; unfold[0,2]}", None, 17))
    return cases


def config_cases():
    """Appendix-A config operators at reduced sizes, with batch."""
    small = {"C_out": 5, "C_in": 4, "H": 6, "W": 7, "K": 3, "N": 2}
    cases = [
        ("conv3x3", conv_spec(small), CONV_STEPS, None, 21),
        ("conv3x3_s2", conv_spec({**small, "s": 2}, s2=True), CONV_S2, None, 22),
        ("sep_shared", conv_spec(small), SEP_SHARED, None, 23),
        ("pointwise", conv_spec(small), POINTWISE, None, 24),
        ("sumpool3x3", conv_spec({"C": 3, "H": 6, "W": 5, "K": 3, "N": 2}, same_c=True), SUMPOOL, None, 25),
        ("qkv", spec("qkv", ("T", "E", "E3", "B"), (), {"T": 8, "E": 6, "E3": 10, "B": 2},
                     ("T", "E3"), ("T", "E"), ("B",)), QKV, None, 26),
        ("conv3x3_k5", conv_spec({**small, "K": 5}), CONV_STEPS, None, 27),
        # the cfg1 operator under a reduced assignment (same document, assignment argument)
        ("cfg1_reduced", conv_spec({"C_out": 64, "C_in": 64, "H": 32, "W": 32, "K": 3, "N": 8}), CONV_STEPS,
         {"C_out": 3, "C_in": 2, "H": 5, "W": 4, "K": 3, "N": 2}, 28),
    ]
    return cases


def corpus_cases(limit=48):
    path = os.path.join(HERE, "corpus_conv64.txt")
    if not os.path.exists(path):
        return []
    ops = [ln.strip() for ln in open(path) if ln.strip()]
    full = {"C_out": 64, "C_in": 64, "H": 32, "W": 32, "K": 3, "s": 2, "N": 8}
    sp = spec("conv64", ("C_out", "C_in", "H", "W", "N"), ("K", "s"), full,
              ("C_out", "H", "W"), ("C_in", "H", "W"), ("N",))
    reduced_opts = [
        {"C_out": 4, "C_in": 4, "H": 4, "W": 4, "K": 3, "s": 2, "N": 2},
        {"C_out": 2, "C_in": 4, "H": 8, "W": 4, "K": 3, "s": 2, "N": 2},
        {"C_out": 4, "C_in": 2, "H": 4, "W": 8, "K": 3, "s": 2, "N": 2},
    ]
    cases = []
    for k, op in enumerate(ops):
        g = parse_steps(op, sp)
        for red in reduced_opts:
            try:
                fl = C.flops(g, red)
                if fl * 4 > 3e7:  # keep the reference's full-grid interpreter cheap
                    continue
                C.weight_shapes(g, red)
            except (NonIntegralSize, ValueError):
                continue
            cases.append((f"corpus{k:04d}", sp, op, red, 1000 + k))
            break
        if len(cases) >= limit:
            break
    return cases


def main():
    out_cases = []
    arrays = {}
    for name, sp, steps, assignment, seed in reference_fixture_cases() + config_cases() + corpus_cases():
        g = parse_steps(steps, sp)
        env = dict(assignment) if assignment is not None else dict(sp.reference)
        nest = C.build_loop_nest(g, env)
        staged = C.rfactor(nest)
        rng = np.random.default_rng(seed)
        xshape = C.input_shape(sp, env)
        yshape = C.output_shape(sp, env)
        x = rng.standard_normal(xshape)
        ws = C.random_weights(g, rng, env)
        up = rng.standard_normal(yshape)
        y = C.interpret(g, x, ws, env)
        ys = C.interpret(g, x, ws, env, staged=True)
        dws = C.weight_gradient(g, x, up, ws, env) if ws else []
        out_cases.append({
            "name": name,
            "document": print_operator(g),
            "steps": steps,
            "assignment": assignment,
            "env": env,
            "batch_shape": [int(v) for v in xshape[: len(sp.batch_dims)]],
            "nest": C.emit_loop_nest(nest),
            "nest_staged": C.emit_loop_nest(staged),
            "n_stages": len(staged.stages),
            "flops": int(C.flops(g, env)),
            "flops_staged": int(C.flops(g, env, staged=True)),
            "params": int(C.param_count(g, env)),
            "n_weights": len(ws),
        })
        arrays[f"{name}/x"] = x
        arrays[f"{name}/up"] = up
        arrays[f"{name}/y"] = y
        arrays[f"{name}/y_staged"] = ys
        for j, (w, dw) in enumerate(zip(ws, dws)):
            arrays[f"{name}/w{j}"] = w
            arrays[f"{name}/dw{j}"] = dw
        print(name, "ok", len(staged.stages), "stages", flush=True)
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(out_cases, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "tensors.npz"), **arrays)
    print(len(out_cases), "cases")


if __name__ == "__main__":
    main()

"""Golden shape distances from the REFERENCE (opsmith.shapedist).

Test infrastructure only: imports the read-only reference from
/root/reference/pkg/src (this container only) and writes
tests/golden/shapedist.json, which tests/test_shapedist.py compares with
the native solver (csrc/shapedist.cpp via paper_2410_23745_b200.shapedist).

Three families:
  * "problems": seeded random frontiers (sizes over the conv2d/strided
    variables with negative coefficient exponents, reduce-pure / strided
    flags) against random input dims, both may_reduce readings
    (shape_distance, shapedist.py:405-412);
  * "tree": 4000 seeded distinct nodes of the complete unpruned step tree
    of the vec1d spec to depth 4 and of the conv2d spec to depth 3 (the
    reference's own admissibility fixture, tests/test_shapedist.py:164-245),
    replayed from their step strings (graph_distance, shapedist.py:415-420);
  * "corpus": every prefix of the first 160 corpus operators on the conv64
    spec (graph_distance).

    python tests/golden/make_shapedist.py
"""
from __future__ import annotations

import json
import os
import random
import sys

sys.path.insert(0, "/root/reference/pkg/src")

from opsmith.pgraph import ProblemSpec, apply, parse_steps, print_steps, root  # noqa: E402
from opsmith.search import legal_steps  # noqa: E402
from opsmith.shapedist import DimDesc, graph_distance, shape_distance  # noqa: E402
from opsmith.symexpr import Variable, parse_size  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def build_spec(name, primaries, coeffs, reference, output, input_, batch=()):
    variables = tuple(Variable(n) for n in primaries) + tuple(Variable(n, primary=False) for n in coeffs)
    vm = {v.name: v for v in variables}
    return ProblemSpec(name=name, variables=variables, reference=tuple(reference.items()),
                       output_dims=tuple(parse_size(t, vm) for t in output),
                       input_dims=tuple(parse_size(t, vm) for t in input_),
                       batch_dims=tuple(parse_size(t, vm) for t in batch))


SPECS = {
    "vec1d": (("vecmap", ("N",), ("g",), {"N": 8, "g": 2}, ("N",), ("N",)), 4),
    "conv2d": (("conv2d", ("C_out", "C_in", "H", "W"), ("K",), {"C_out": 8, "C_in": 8, "H": 8, "W": 8, "K": 3},
                ("C_out", "H", "W"), ("C_in", "H", "W")), 3),
}
CORPUS_SPEC = ("conv64", ("C_out", "C_in", "H", "W", "N"), ("K", "s"),
               {"C_out": 64, "C_in": 64, "H": 32, "W": 32, "K": 3, "s": 2, "N": 8},
               ("C_out", "H", "W"), ("C_in", "H", "W"), ("N",))


def size_text(rng, vm):
    prim = ["C_out", "C_in", "H", "W"]
    coef = ["K", "s"]
    parts = []
    for name in rng.sample(prim, rng.choice([0, 1, 1, 1, 2])):
        parts.append(name if rng.random() < 0.8 else f"{name}^2")
    for name in rng.sample(coef, rng.choice([0, 0, 1, 2])):
        e = rng.choice([1, 1, -1, 2])
        parts.append(name if e == 1 else f"{name}^{e}")
    if not parts:
        return "1"
    return "*".join(sorted(parts, key=lambda p: p.split("^")[0]))


def problems(n=1500, seed=11):
    spec = build_spec("strided", ("C_out", "C_in", "H", "W"), ("K", "s"),
                      {"C_out": 4, "C_in": 4, "H": 8, "W": 8, "K": 3, "s": 2}, ("C_out", "H", "W"), ("C_in", "H", "W"))
    vm = spec.var_map
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        cur = []
        for _ in range(rng.randint(0, 5)):
            cur.append((size_text(rng, vm), rng.random() < 0.3, rng.random() < 0.2))
        tgt = [size_text(rng, vm) for _ in range(rng.randint(0, 3))]
        if rng.random() < 0.5:
            tgt = ["C_in", "H", "W"][: rng.randint(1, 3)]
        descs = [DimDesc(parse_size(t, vm), pure, st) for t, pure, st in cur]
        sizes = [parse_size(t, vm) for t in tgt]
        d0 = shape_distance(descs, sizes, may_reduce=False)
        d1 = shape_distance(descs, sizes, may_reduce=True)
        out.append({"current": cur, "inputs": tgt, "d": [d0, d1]})
    return out


def tree(args, depth):
    spec = build_spec(*args)
    nodes = [root(spec)]
    start = 0
    for _ in range(depth):
        end = len(nodes)
        for i in range(start, end):
            for step in legal_steps(nodes[i]):
                nodes.append(apply(nodes[i], step))
        start = end
    seen = {}
    for g in nodes:
        seen.setdefault(print_steps(g), graph_distance(g))
    rows = [{"steps": k, "d": v} for k, v in seen.items()]
    return random.Random(5).sample(rows, min(len(rows), 4000))


def corpus(limit=160):
    spec = build_spec(*CORPUS_SPEC)
    ops = [ln.strip() for ln in open(os.path.join(HERE, "corpus_conv64.txt")) if ln.strip()][:limit]
    seen = {}
    for op in ops:
        body = [p.strip() for p in op[3:-1].split(";")]
        for k in range(len(body) + 1):
            text = "op{" + "; ".join(body[:k]) + "}"
            if text not in seen:
                seen[text] = graph_distance(parse_steps(text, spec))
    return [{"steps": k, "d": v} for k, v in seen.items()]


def enc(v):
    return "inf" if v == float("inf") else v


def main():
    out = {"problems": problems(), "trees": {}, "corpus": corpus(), "specs": {k: v[0] for k, v in SPECS.items()},
           "corpus_spec": CORPUS_SPEC}
    for name, (args, depth) in SPECS.items():
        out["trees"][name] = tree(args, depth)
    for p in out["problems"]:
        p["d"] = [enc(v) for v in p["d"]]
    for rows in list(out["trees"].values()) + [out["corpus"]]:
        for r in rows:
            r["d"] = enc(r["d"])
    with open(os.path.join(HERE, "shapedist.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print({"problems": len(out["problems"]), "corpus": len(out["corpus"]),
           **{k: len(v) for k, v in out["trees"].items()}})


if __name__ == "__main__":
    main()

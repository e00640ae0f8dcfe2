"""Native shape distance (csrc/shapedist.cpp) against the reference.

The reference's own unit tests (pkg/tests/test_shapedist.py:32-161) are
restated on this package's API, then the golden distances the reference
itself computed (tests/golden/make_shapedist.py) are compared value for
value: random frontiers, nodes of the complete step trees (the reference's
admissibility fixture) and every prefix of 160 corpus operators.  When the
reference tree is present (this container) a live comparison on fresh
random problems runs as well.
"""
from __future__ import annotations

import json
import os
import random
import sys

import pytest

from paper_2410_23745_b200 import shapedist as SD
from paper_2410_23745_b200.pgraph import build_spec, parse_steps
from paper_2410_23745_b200.shapedist import INF, DimDesc, ReshapeGroup

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "shapedist.json")
CONV_STEPS = ("op{reduce(C_in); reduce(K); reduce(K); "
              "contract[0:weight,3:both,4:both,5:both]; unfold[1,7]; unfold[2,8]}")
CONV_INPUT = ("C_in", "H", "W")


def conv2d():
    return build_spec("conv2d", ("C_out", "C_in", "H", "W"), ("K",),
                      {"C_out": 8, "C_in": 8, "H": 8, "W": 8, "K": 3}, ("C_out", "H", "W"), CONV_INPUT)


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def dec(v):
    return INF if v == "inf" else v


# ---- the reference's unit tests (pkg/tests/test_shapedist.py) on this API ----

def test_group_cost_values():
    balanced = ReshapeGroup(("H*s^-1", "W*s"), ("H", "W"))
    assert not balanced.needs_elimination
    assert SD.group_cost(balanced) == 2
    assert SD.group_cost(ReshapeGroup(("C_in",), ("C_in",))) == 0
    eliminate = ReshapeGroup(("k",), ())
    assert eliminate.needs_elimination
    assert SD.group_cost(eliminate) == 1


def test_worked_strided_distance():
    current = [DimDesc("C_in"), DimDesc("H*s^-1"), DimDesc("W*s", strided=True), DimDesc("k", reduce_pure=True)]
    target = ["C_in", "H", "W"]
    assert SD.shape_distance(current, target, may_reduce=False) == 3
    result = SD.explain_distance(current, target, may_reduce=False)
    assert result.distance == 3
    covered = [size for g in result.groups for size in g.rhs]
    assert sorted(map(str, covered)) == sorted(target)
    # the witness is a partition whose group costs are admissible pieces of the total
    assert sorted(str(d) for g in result.groups for d in g.lhs) == sorted(str(d.size) for d in current)


def test_window_eliminations_cost_one_each():
    current = [DimDesc("C_in"), DimDesc("H"), DimDesc("W"), DimDesc("K", True), DimDesc("K", True)]
    assert SD.shape_distance(current, CONV_INPUT) == 2


def test_bundled_elimination_costs_one_total():
    current = [DimDesc(s) for s in ("C_in", "H", "W", "C_out", "C_out")]
    assert SD.shape_distance(current, CONV_INPUT) == 1


def test_deficit_repair_via_stride():
    assert SD.shape_distance([DimDesc("H*s^-1"), DimDesc("k", reduce_pure=True)], ["H"], may_reduce=False) == 2


def test_creation_needs_reduction_stage():
    assert SD.shape_distance([], ["C_in"], may_reduce=False) == INF
    assert SD.shape_distance([], ["C_in"], may_reduce=True) == 1


def test_conv2d_progression():
    spec = conv2d()
    assert SD.graph_distance(parse_steps("op{}", spec)) == 2
    assert SD.graph_distance(parse_steps("op{reduce(C_in)}", spec)) == 1
    assert SD.graph_distance(parse_steps(CONV_STEPS, spec)) == 0
    # frontier of the finished conv is (C_in, H, W) in input order
    result = SD.explain_distance([DimDesc(s) for s in CONV_INPUT], CONV_INPUT)
    assert result.permutation == (0, 1, 2)


def test_distance_zero_iff_matchable():
    sizes = ["C_in", "H", "W", "C_out", "K"]
    rng = random.Random(7)
    for _ in range(80):
        picked = [rng.choice(sizes) for _ in range(rng.randint(1, 4))]
        strided = [rng.random() < 0.2 for _ in picked]
        current = [DimDesc(sz, strided=st) for sz, st in zip(picked, strided)]
        d = SD.shape_distance(current, CONV_INPUT)
        matchable = sorted(picked) == sorted(CONV_INPUT) and not any(strided)
        assert (d == 0) == matchable, (picked, strided, d)


def test_distance_is_permutation_invariant():
    current = [DimDesc("W*s", strided=True), DimDesc("k", reduce_pure=True), DimDesc("C_in"), DimDesc("H*s^-1")]
    target = ["C_in", "H", "W"]
    rng = random.Random(3)
    want = SD.shape_distance(current, target)
    for _ in range(10):
        rng.shuffle(current)
        assert SD.shape_distance(current, target) == want


def test_strided_dim_alone_is_never_distance_zero():
    current = [DimDesc("C_in", strided=True), DimDesc("H"), DimDesc("W")]
    assert SD.shape_distance(current, CONV_INPUT) >= 1


def test_cache_clear_keeps_answers():
    current = [DimDesc("C_in"), DimDesc("H*s^-1"), DimDesc("W*s", strided=True), DimDesc("k", reduce_pure=True)]
    a = SD.shape_distance(current, CONV_INPUT)
    SD.clear_cache()
    assert SD.shape_distance(current, CONV_INPUT) == a


# ---- golden values the reference computed ----

def test_random_problems_match_reference(golden):
    for p in golden["problems"]:
        cur = [DimDesc(s, pure, st) for s, pure, st in p["current"]]
        for may_reduce, want in zip((False, True), p["d"]):
            got = SD.shape_distance(cur, p["inputs"], may_reduce=may_reduce)
            assert got == dec(want), (p, may_reduce, got)


def test_explain_distance_witness_is_optimal(golden):
    """The witness partitions both sides and its distance is the reference's."""
    for p in golden["problems"][:400]:
        cur = [DimDesc(s, pure, st) for s, pure, st in p["current"]]
        r = SD.explain_distance(cur, p["inputs"], may_reduce=True)
        assert r.distance == dec(p["d"][1])
        if r.distance == INF:
            continue
        assert sorted(str(s) for g in r.groups for s in g.rhs) == sorted(p["inputs"])
        assert len([s for g in r.groups for s in g.lhs]) == len(cur)


@pytest.mark.parametrize("tree", ["vec1d", "conv2d"])
def test_step_tree_graph_distances_match_reference(golden, tree):
    spec = build_spec(*golden["specs"][tree])
    for row in golden["trees"][tree]:
        g = parse_steps(row["steps"], spec)
        assert SD.graph_distance(g) == dec(row["d"]), row


def test_corpus_prefix_graph_distances_match_reference(golden):
    spec = build_spec(*golden["corpus_spec"])
    for row in golden["corpus"]:
        assert SD.graph_distance(parse_steps(row["steps"], spec)) == dec(row["d"]), row


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree absent (GPU box)")
def test_live_against_reference_objects():
    """Fresh random problems on the reference's own SymbolicSize objects, and
    graph_distance of reference PGraphs, against the reference itself."""
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from opsmith import shapedist as RSD
    from opsmith.pgraph import ProblemSpec, parse_steps as ref_parse
    from opsmith.symexpr import Variable, parse_size

    variables = tuple(Variable(n) for n in ("C_out", "C_in", "H", "W")) + tuple(
        Variable(n, primary=False) for n in ("K", "s"))
    vm = {v.name: v for v in variables}
    rng = random.Random(2024)
    names = ["C_out", "C_in", "H", "W", "K", "s^-1", "s", "K^2", "H*s^-1", "W*s", "C_in*K"]
    for _ in range(300):
        cur = [RSD.DimDesc(parse_size(rng.choice(names), vm), rng.random() < 0.3, rng.random() < 0.2)
               for _ in range(rng.randint(0, 6))]
        tgt = [parse_size(rng.choice(names[:4]), vm) for _ in range(rng.randint(0, 3))]
        mine = [DimDesc(d.size, d.reduce_pure, d.strided) for d in cur]
        for mr in (False, True):
            assert SD.shape_distance(mine, tgt, mr) == RSD.shape_distance(cur, tgt, mr)
    spec = ProblemSpec(name="conv2d", variables=variables[:4] + variables[4:5],
                       reference=(("C_out", 8), ("C_in", 8), ("H", 8), ("W", 8), ("K", 3)),
                       output_dims=tuple(parse_size(t, vm) for t in ("C_out", "H", "W")),
                       input_dims=tuple(parse_size(t, vm) for t in CONV_INPUT))
    for text in ("op{}", "op{reduce(C_in)}", "op{reduce(C_in); reduce(K)}", CONV_STEPS):
        g = ref_parse(text, spec)
        assert SD.graph_distance(g) == RSD.graph_distance(g)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree absent (GPU box)")
def test_reference_search_log_unchanged_with_native_distance(monkeypatch):
    """INTEGRATION.md's search-side opt-in: the reference's own MCTS with
    graph_distance swapped for the native one logs the same samples, byte
    for byte, for the same seed (search.py:62, 166-171)."""
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import numpy as np
    import opsmith.search as S
    from opsmith.pgraph import ProblemSpec, print_steps
    from opsmith.symexpr import Variable, parse_size

    variables = (Variable("C_out"), Variable("C_in"), Variable("H"), Variable("W"), Variable("K", primary=False))
    vm = {v.name: v for v in variables}
    spec = ProblemSpec(name="conv2d", variables=variables,
                       reference=(("C_out", 8), ("C_in", 8), ("H", 8), ("W", 8), ("K", 3)),
                       output_dims=tuple(parse_size(t, vm) for t in ("C_out", "H", "W")),
                       input_dims=tuple(parse_size(t, vm) for t in ("C_in", "H", "W")))

    def reward(g):
        return (sum(map(ord, print_steps(g))) % 97) / 97.0

    def run():
        tree = S.SearchTree(spec, S.Budget(d_max=7), seed=11)
        rng = np.random.default_rng(11)
        return [r.line() for r in (S.mcts_step(tree, reward, rng) for _ in range(300)) if r is not None]

    want = run()
    monkeypatch.setattr(S, "graph_distance", SD.graph_distance)
    got = run()
    assert want and got == want

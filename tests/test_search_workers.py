"""Multi-GPU search workers on the reference's own MCTS (CPU).

The reference search (opsmith.search, /root/reference/pkg/src) is driven
through ``search_workers.run_workers`` with a host reward (the device reward
is covered by tests/test_gpu_search_workers.py): one worker reproduces the
reference's sequential log byte for byte (test_search.py:208-214); several
workers share the tree, take exactly the requested iterations and log
unique, dense sample ids in the reference grammar.
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
    import opsmith.search as S
    from opsmith.pgraph import ProblemSpec
    from opsmith.symexpr import Variable, parse_size
    variables = (Variable("C_out"), Variable("C_in"), Variable("H"), Variable("W"), Variable("K", primary=False))
    vm = {v.name: v for v in variables}
    spec = ProblemSpec(name="conv2d", variables=variables,
                       reference=(("C_out", 8), ("C_in", 8), ("H", 8), ("W", 8), ("K", 3)),
                       output_dims=tuple(parse_size(t, vm) for t in ("C_out", "H", "W")),
                       input_dims=tuple(parse_size(t, vm) for t in ("C_in", "H", "W")))
    return S, spec


def _reward(g):
    # a deterministic host reward that depends on the operator
    from opsmith.pgraph import print_steps
    return (sum(map(ord, print_steps(g))) % 97) / 97.0


def test_one_worker_reproduces_the_reference_log(ref):
    import numpy as np

    from paper_2410_23745_b200.search_workers import run_workers
    S, spec = ref
    t1 = S.SearchTree(spec, S.Budget(d_max=6), seed=7)
    rng = np.random.default_rng(7)
    want = [r.line() for r in (S.mcts_step(t1, _reward, rng) for _ in range(120)) if r is not None]
    t2 = S.SearchTree(spec, S.Budget(d_max=6), seed=7)
    got = [r.line() for r in run_workers(t2, S.mcts_step, [_reward], 120, [7])]
    assert want and got == want


def test_several_workers_share_one_tree(ref):
    from paper_2410_23745_b200.search_workers import run_workers
    S, spec = ref
    tree = S.SearchTree(spec, S.Budget(d_max=6), seed=3)
    recs = run_workers(tree, S.mcts_step, [_reward] * 4, 200, [3, 4, 5, 6])
    assert tree.iteration == 200
    ids = [r.sample_id for r in recs]
    assert ids == list(range(len(ids))) and ids
    for r in recs:
        assert S.parse_record(r.line()) == r
    # virtual loss is fully released: no node keeps a pending visit
    stack = [tree.root]
    while stack:
        n = stack.pop()
        assert n.virtual == 0
        stack.extend(n.children.values())


def test_worker_errors_surface(ref):
    from paper_2410_23745_b200.search_workers import run_workers
    S, spec = ref

    def boom(g):
        raise ZeroDivisionError("reward backend crashed")
    tree = S.SearchTree(spec, S.Budget(d_max=6), seed=1)
    with pytest.raises(ZeroDivisionError):
        run_workers(tree, S.mcts_step, [boom, boom], 50, [1, 2])
    with pytest.raises(ValueError):
        run_workers(tree, S.mcts_step, [boom], 5, [1, 2])

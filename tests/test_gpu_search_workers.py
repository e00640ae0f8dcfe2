"""GPU: the reference's MCTS driven by device-reward workers.

The reference package comes from baseline/_ref (the pip --target install
that travels to the GPU box; skipped when absent).  The reward is the
device-resident fit reward (reward.builtin_fit_reward on the GPU, float64)
toward the reference's conv2d target (tests/golden/rewards.json's spec).
Checks: equal seeds give byte-identical logs with the device reward in the
loop (the reference contract, test_search.py:208-214 -- it needs the
deterministic scatter); several workers share one tree and every logged
reward equals a fresh single-call evaluation of the same operator.
"""
from __future__ import annotations

import functools
import json
import os
import sys

import pytest

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu


def _opsmith():
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "opsmith")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import opsmith.search as S
            from opsmith.pgraph import ProblemSpec
            from opsmith.symexpr import Variable, parse_size
            return S, ProblemSpec, Variable, parse_size
    pytest.skip("reference package not installed (baseline/_ref)")


@pytest.fixture(scope="module")
def setup(cuda):
    S, ProblemSpec, Variable, parse_size = _opsmith()
    from paper_2410_23745_b200 import reward as R
    from paper_2410_23745_b200.pgraph import build_spec
    with open(os.path.join(GOLDEN, "rewards.json")) as f:
        G = json.load(f)
    sp = G["spec"]
    variables = tuple(Variable(n) for n in sp["primaries"]) + tuple(Variable(n, primary=False) for n in sp["coeffs"])
    vm = {v.name: v for v in variables}
    ref_spec = ProblemSpec(name=sp["name"], variables=variables, reference=tuple(sp["reference"].items()),
                           output_dims=tuple(parse_size(t, vm) for t in sp["output"]),
                           input_dims=tuple(parse_size(t, vm) for t in sp["input_"]))
    target = R.fit_target(build_spec(**sp), G["target"], seed=G["target_seed"], samples=G["samples"])
    return S, ref_spec, target


def _fn(target):
    from paper_2410_23745_b200 import reward as R
    return R.make_reward_fn(functools.partial(R.builtin_fit_reward, target=target))


def test_device_reward_search_is_deterministic(setup):
    from paper_2410_23745_b200.search_workers import run_workers
    S, spec, target = setup
    logs = []
    for _ in range(2):
        tree = S.SearchTree(spec, S.Budget(d_max=5), seed=11)
        logs.append([r.line() for r in run_workers(tree, S.mcts_step, [_fn(target)], 40, [11], devices=[0])])
    assert logs[0] and logs[0] == logs[1]


def test_workers_share_the_tree_with_device_rewards(setup):
    from paper_2410_23745_b200 import reward as R
    from paper_2410_23745_b200.search_workers import run_workers
    S, spec, target = setup
    tree = S.SearchTree(spec, S.Budget(d_max=5), seed=5)
    recs = run_workers(tree, S.mcts_step, [_fn(target), _fn(target)], 40, [5, 6], devices=[0, 0])
    assert tree.iteration == 40
    assert [r.sample_id for r in recs] == list(range(len(recs)))
    for r in recs:
        if r.status != "ok":
            continue
        from opsmith.pgraph import parse_steps
        again = R.builtin_fit_reward(parse_steps(r.op, tree.spec), target).reward
        assert r.reward == min(1.0, max(0.0, again))

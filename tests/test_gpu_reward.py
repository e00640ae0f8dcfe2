"""GPU: the device-resident fit reward against the REFERENCE's own values.

tests/golden/rewards.json was produced by reward.builtin_fit_reward of the
reference (tests/golden/make_rewards.py); the cases mirror the reference's
tests (pkg/tests/test_reward.py:44-63: the target fits itself >= 0.99 with
residual < 1e-8; the partial conv scores ~0.599).  LSQR runs on the device
in float64 with the backend's forward / weight-gradient kernels as matvec /
rmatvec; the converged fits agree with scipy's to 1e-6 in the reward.
"""
from __future__ import annotations

import json
import os

import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _golden():
    with open(os.path.join(GOLDEN, "rewards.json")) as f:
        return json.load(f)


G = _golden()


@pytest.fixture(scope="module")
def target(cuda):
    from paper_2410_23745_b200 import reward as R
    from paper_2410_23745_b200.pgraph import build_spec
    spec = build_spec(**G["spec"])
    return spec, R.fit_target(spec, G["target"], seed=G["target_seed"], samples=G["samples"])


def test_target_energy_matches_reference(target):
    _, t = target
    assert t.norm == pytest.approx(G["target_norm"], rel=1e-12)


@pytest.mark.parametrize("case", G["cases"], ids=[f"{c['name']}-s{c['seed']}" for c in G["cases"]])
def test_fit_reward_matches_reference(target, case):
    from paper_2410_23745_b200 import reward as R
    from paper_2410_23745_b200.pgraph import parse_steps
    spec, t = target
    rep = R.builtin_fit_reward(parse_steps(case["steps"], spec), t, seed=case["seed"])
    assert rep.reward == pytest.approx(case["reward"], abs=1e-6)
    assert rep.diag("weights") == case["weights"]
    if case["name"] == "self":
        assert rep.reward >= 0.99 and float(rep.diag("residual")) < 1e-8


def test_reward_fn_memoises(target):
    from paper_2410_23745_b200 import reward as R
    from paper_2410_23745_b200.pgraph import parse_steps
    spec, t = target
    calls = []

    def backend(g):
        calls.append(g)
        return R.builtin_fit_reward(g, t)

    fn = R.make_reward_fn(backend)
    g = parse_steps(G["cases"][0]["steps"], spec)
    assert fn(g) == fn(g)
    assert len(calls) == 1


@pytest.mark.parametrize("name", ["self", "partial"])
def test_external_protocol_child(cuda, name):
    """The GPU reward child speaks the reference's external-reward protocol
    (reward.py:179-222): operator document on stdin, `reward <float>` and
    `diag k v` lines on stdout."""
    import subprocess
    import sys

    from conftest import ROOT
    from paper_2410_23745_b200.pgraph import build_spec, parse_steps
    case = next(c for c in G["cases"] if c["name"] == name and c["seed"] == 0)
    spec = build_spec(**G["spec"])
    doc = parse_steps(case["steps"], spec).document
    r = subprocess.run([sys.executable, "-m", "paper_2410_23745_b200.reward_child", "--target", G["target"],
                        "--seed", "0"], input=doc, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    head = lines[0].split()
    assert head[0] == "reward" and float(head[1]) == pytest.approx(case["reward"], abs=1e-6)
    assert any(ln.startswith("diag residual ") for ln in lines[1:])

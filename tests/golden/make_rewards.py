"""Golden fit-reward values from the REFERENCE (reward.builtin_fit_reward).

Test infrastructure only: imports the read-only reference from
/root/reference/pkg/src (this container only) and writes
tests/golden/rewards.json, which tests/test_gpu_reward.py compares with the
device-resident reward (paper_2410_23745_b200/reward.py).

Cases follow the reference's own tests (pkg/tests/test_reward.py:21-76):
the conv target on the small conv spec, candidates = the target itself,
the partial conv, a two-weight shared-kernel op and a
pointwise op, at two seeds.

    python tests/golden/make_rewards.py
"""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")

from opsmith.pgraph import ProblemSpec, parse_steps  # noqa: E402
from opsmith.reward import builtin_fit_reward, fit_target  # noqa: E402
from opsmith.symexpr import Variable, parse_size  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

SPEC = dict(name="conv2d", primaries=("C_out", "C_in", "H", "W"), coeffs=("K",),
            reference={"C_out": 3, "C_in": 2, "H": 5, "W": 5, "K": 3},
            output=("C_out", "H", "W"), input_=("C_in", "H", "W"))

CONV = ("op{reduce(C_in); reduce(K); reduce(K); contract[0:weight,3:both,4:both,5:both]; "
        "unfold[1,7]; unfold[2,8]}")
CANDIDATES = {
    "self": CONV,
    "partial": "op{reduce(C_in); reduce(K); contract[0:weight,3:both,4:both]; unfold[1,6]}",
    "sep_shared": ("op{reduce(C_in); reduce(K); reduce(K); contract[0:weight,3:both,4:both]; "
                   "unfold[1,7]; contract[5:both]; unfold[2,9]}"),
    "pointwise": "op{reduce(C_in); contract[0:weight,3:both]}",
}


def ref_spec():
    variables = tuple(Variable(n) for n in SPEC["primaries"]) + tuple(Variable(n, primary=False)
                                                                      for n in SPEC["coeffs"])
    vm = {v.name: v for v in variables}
    return ProblemSpec(name=SPEC["name"], variables=variables, reference=tuple(SPEC["reference"].items()),
                       output_dims=tuple(parse_size(t, vm) for t in SPEC["output"]),
                       input_dims=tuple(parse_size(t, vm) for t in SPEC["input_"]))


def main():
    spec = ref_spec()
    target = fit_target(spec, CONV, seed=0, samples=2)
    out = {"spec": SPEC, "target": CONV, "target_seed": 0, "samples": 2, "target_norm": target.norm, "cases": []}
    for name, steps in CANDIDATES.items():
        g = parse_steps(steps, spec)
        for seed in (0, 3):
            rep = builtin_fit_reward(g, target, seed=seed)
            out["cases"].append({"name": name, "steps": steps, "seed": seed, "reward": rep.reward,
                                 "residual": rep.diag("residual"), "weights": rep.diag("weights")})
            print(name, seed, rep.reward, rep.diag("residual"))
    with open(os.path.join(HERE, "rewards.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

"""GPU reward child for the reference's external-reward protocol.

The reference's ``external_reward(graph, command)`` (reward.py:179-222)
writes the operator document to a child's stdin and reads one line
``reward <float>`` plus optional ``diag <key> <value>`` lines from its
stdout; timeouts, non-zero exits and unparseable output become
``RewardFailure``.  This module is such a child, backed by the device-
resident fit reward (reward.builtin_fit_reward on the B200):

    external_reward(graph, "python -m paper_2410_23745_b200.reward_child --target 'op{...}' --seed 0")

The target operator is given as a step string over the candidate's own
spec (the document's header), as reward.fit_target takes it.  Exit codes:
0 ok, 2 bad input (the parent turns both non-zero codes into a failure).
"""
from __future__ import annotations

import argparse
import sys

CONV_TARGET = ("op{reduce(C_in); reduce(K); reduce(K); contract[0:weight,3:both,4:both,5:both]; "
               "unfold[1,7]; unfold[2,8]}")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="reward_child")
    ap.add_argument("--target", default=CONV_TARGET, help="target operator steps over the candidate's spec")
    ap.add_argument("--seed", type=int, default=0, help="fit seed (reward.builtin_fit_reward)")
    ap.add_argument("--target-seed", type=int, default=0)
    ap.add_argument("--samples", type=int, default=2)
    args = ap.parse_args(argv)
    doc = sys.stdin.read()

    from .errors import GraphError, OperatorParseError
    from .pgraph import parse_operator
    from .reward import builtin_fit_reward, fit_target
    try:
        graph = parse_operator(doc)
        target = fit_target(graph.spec, args.target, seed=args.target_seed, samples=args.samples)
    except (OperatorParseError, GraphError, ValueError, KeyError) as exc:
        print(f"bad operator document: {exc}", file=sys.stderr)
        return 2
    report = builtin_fit_reward(graph, target, seed=args.seed)
    print(f"reward {report.reward!r}")
    for k, v in report.diagnostics:
        print(f"diag {k} {v}")
    return 0


if __name__ == "__main__":
    sys.exit(main())

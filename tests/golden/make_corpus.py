"""Generate the cfg5 candidate corpus with the REFERENCE sampler.

Test/bench infrastructure only: imports the read-only reference from
/root/reference/pkg/src (this container only) and writes the sampled
step strings to tests/golden/corpus_conv64.txt.  The GPU box never runs
this script; it only reads the committed text file.

Sampler: ``opsmith.search.random_completion`` (search.py:562-574) on a
batch-free conv spec {C_in=C_out=64, H=W=32, K=3, s=2}, d_max=7,
flops_cap = 10x the dense conv3x3, fixed seeds.

    python tests/golden/make_corpus.py [count] [seconds]
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from opsmith.pgraph import ProblemSpec, print_steps  # noqa: E402
from opsmith.search import SearchTree, random_completion  # noqa: E402
from opsmith.symexpr import Variable, parse_size  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def conv_spec(flops_cap):
    variables = (
        Variable("C_out"), Variable("C_in"), Variable("H"), Variable("W"),
        Variable("K", primary=False), Variable("s", primary=False),
    )
    vm = {v.name: v for v in variables}
    ref = (("C_out", 64), ("C_in", 64), ("H", 32), ("W", 32), ("K", 3), ("s", 2))
    return ProblemSpec(
        name="conv64",
        variables=variables,
        reference=ref,
        output_dims=tuple(parse_size(t, vm) for t in ("C_out", "H", "W")),
        input_dims=tuple(parse_size(t, vm) for t in ("C_in", "H", "W")),
        max_depth=7,
        flops_cap=flops_cap,
        params_cap=64 * 64 * 9 * 16,
    )


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    budget_s = float(sys.argv[2]) if len(sys.argv) > 2 else 3000.0
    conv_flops = 2 * 64 * 32 * 32 * 64 * 9
    spec = conv_spec(10 * conv_flops)
    out_path = os.path.join(HERE, "corpus_conv64.txt")
    seen = set()
    ops = []
    seed = 0
    t0 = time.time()
    while len(ops) < count and time.time() - t0 < budget_s:
        tree = SearchTree(spec, seed=seed)
        g = random_completion(tree, np.random.default_rng(seed))
        seed += 1
        if g is None:
            continue
        text = print_steps(g)
        if text in seen:
            continue
        seen.add(text)
        ops.append(text)
        if len(ops) % 32 == 0:
            with open(out_path, "w") as f:
                f.write("\n".join(ops) + "\n")
            print(len(ops), "ops", f"{time.time() - t0:.0f}s", flush=True)
    with open(out_path, "w") as f:
        f.write("\n".join(ops) + "\n")
    print("done", len(ops), "ops from", seed, "seeds", f"{time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()

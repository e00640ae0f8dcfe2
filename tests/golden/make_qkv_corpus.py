"""Sampled variants of the GPT-2-small QKV projection
with the REFERENCE sampler.

Test/bench infrastructure only: imports the read-only reference from
/root/reference/pkg/src (this container only) and writes the sampled
step strings to tests/golden/corpus_qkv.txt; the GPU box reads the file.

Sampler: ``opsmith.search.random_completion`` (search.py:562-574) on the
batch-free QKV spec {T=1024, E=768, E3=2304} (output (T, E3), input (T, E)),
d_max=6, flops_cap = 2x the dense projection, params_cap = 2x its weight,
fixed seeds; only operators with at least one weight are kept (the
projection's sampled replacements), the dense baseline first.

    python tests/golden/make_qkv_corpus.py [count] [seconds]
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from opsmith.codegen import flops, param_count  # noqa: E402
from opsmith.pgraph import ProblemSpec, print_steps  # noqa: E402
from opsmith.search import SearchTree, random_completion  # noqa: E402
from opsmith.symexpr import Variable, parse_size  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DENSE = "op{reduce(E); contract[1:weight,2:both]}"


def qkv_spec(flops_cap, params_cap):
    variables = (Variable("T"), Variable("E"), Variable("E3"))
    vm = {v.name: v for v in variables}
    return ProblemSpec(
        name="qkv",
        variables=variables,
        reference=(("T", 1024), ("E", 768), ("E3", 2304)),
        output_dims=tuple(parse_size(t, vm) for t in ("T", "E3")),
        input_dims=tuple(parse_size(t, vm) for t in ("T", "E")),
        max_depth=6,
        flops_cap=flops_cap,
        params_cap=params_cap,
    )


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    budget_s = float(sys.argv[2]) if len(sys.argv) > 2 else 900.0
    dense_flops = 2 * 1024 * 768 * 2304
    spec = qkv_spec(2 * dense_flops, 2 * 768 * 2304)
    ops, seen = [DENSE], {DENSE}
    seed, t0 = 0, time.time()
    while len(ops) < count and time.time() - t0 < budget_s:
        tree = SearchTree(spec, seed=seed)
        g = random_completion(tree, np.random.default_rng(seed))
        seed += 1
        if g is None or not g.weights:
            continue
        # the search's budget check (search.py:347-356): random_completion does not apply it
        if flops(g) > spec.flops_cap or param_count(g) > spec.params_cap:
            continue
        text = print_steps(g)
        if text in seen:
            continue
        seen.add(text)
        ops.append(text)
        print(len(ops), f"{flops(g) / 1e9:.2f} GFLOP", text, flush=True)
    with open(os.path.join(HERE, "corpus_qkv.txt"), "w") as f:
        f.write("\n".join(ops) + "\n")
    print("done", len(ops), "ops from", seed, "seeds", f"{time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()

"""Multi-GPU search workers.

The reference's ``mcts_step`` (search.py:359-460) holds the tree lock only
for selection / expansion and back-propagation and evaluates the reward
OUTSIDE it, with virtual loss steering concurrent selections apart
(search.py:374-392, 409-440): concurrent evaluation from several threads is
its intended extension point ("Threading").  This module
drives that function from one worker thread per GPU, sharing one tree:

    from opsmith.search import SearchTree, mcts_step
    from paper_2410_23745_b200 import reward as R
    from paper_2410_23745_b200.search_workers import run_workers
    tree = SearchTree(spec, budget, seed=0)
    fns = [R.make_reward_fn(partial(R.builtin_fit_reward, target=t)) for _ in devices]
    records = run_workers(tree, mcts_step, fns, iterations=1000, seeds=[0, 1, ...], devices=[0, 1, ...])

Each worker binds its CUDA device before its first iteration, so every
kernel its reward launches runs there (the native library keeps one device
plan per (operator, device)).  Iterations are claimed from a shared
counter, so the tree sees exactly ``iterations`` steps whatever the worker
count.  With ONE worker the call sequence -- and therefore the log -- is
the reference's sequential loop with ``rng = default_rng(seeds[0])``
(test_search.py:208-214's equal-seeds contract).  With several workers the
interleaving of selections is timing dependent (as in any parallel MCTS);
each logged line still follows the reference grammar (search.py:166-171),
sample ids stay unique and dense, and each operator's reward is
deterministic because the device reward is (fixed-point scatter, DESIGN.md
§3.1).  The reference itself is passed in (``mcts_step``), not imported:
this package does not depend on the search code.
"""
from __future__ import annotations

import threading
from typing import Callable, List, Optional, Sequence


def run_workers(tree, mcts_step: Callable, reward_fns: Sequence[Callable], iterations: int,
                seeds: Sequence[int], devices: Optional[Sequence[int]] = None) -> List:
    """Run ``iterations`` MCTS steps on ``tree`` from ``len(reward_fns)``
    threads; returns the logged records ordered by sample id.  A reward
    failure is logged by the reference before it is raised (the record
    rides on the exception, search.py:455-459); it is kept here and the
    worker carries on."""
    import numpy as np

    n = len(reward_fns)
    if n < 1 or len(seeds) != n or (devices is not None and len(devices) != n):
        raise ValueError("one seed (and one device, when given) per reward function")
    counter = {"next": 0}
    lock = threading.Lock()
    records: List = []
    errors: List[BaseException] = []

    def claim() -> bool:
        with lock:
            if counter["next"] >= iterations:
                return False
            counter["next"] += 1
            return True

    def work(k: int):
        try:
            if devices is not None:
                import torch
                torch.cuda.set_device(devices[k])
            rng = np.random.default_rng(seeds[k])
            while claim():
                try:
                    rec = mcts_step(tree, reward_fns[k], rng)
                except Exception as exc:
                    rec = getattr(exc, "record", None)
                    if rec is None:
                        raise
                if rec is not None:
                    with lock:
                        records.append(rec)
        except BaseException as exc:  # surfaced to the caller after join
            with lock:
                errors.append(exc)

    if n == 1:
        work(0)
    else:
        threads = [threading.Thread(target=work, args=(k,), name=f"syno-search-{k}") for k in range(n)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    if errors:
        raise errors[0]
    records.sort(key=lambda r: r.sample_id)
    return records

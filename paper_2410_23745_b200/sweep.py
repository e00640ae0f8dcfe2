"""Search-time candidate evaluation, sharded one candidate batch per GPU.

The reference evaluates a sampled operator inside ``mcts_step``
(search.py:359-460): ``_score_completion`` computes FLOPs/params and the
budget verdict (search.py:347-356); an over-budget candidate is logged
with status ``over_budget`` and never executed; otherwise ``reward_fn``
runs it (search.py:430-437) and a ``SampleRecord`` line is appended to
the log (search.py:155-171).

Here one *candidate evaluation* is: compile the operator (native lowering
+ plan), run forward, grad-input and every grad-weight on the device on
seeded synthetic inputs, and check the results on the device with two
size-independent identities of a multilinear operator y = A(x; w_1..w_n):

    <dy, y> == <dx, x>          (adjoint of the x access)
    <dy, y> == <dw_j, w_j>      (y is homogeneous of degree 1 in each w_j)

Candidates are independent, so multi-GPU evaluation shards them across
ranks with NO collective on the data path: statically by LPT
on a predicted roofline time (``lpt_shard``), or dynamically -- every rank
claims the next candidate of one shared LPT order from the process group's
key-value store (``StoreClaim``; an atomic counter on the host, no device
traffic).  Each rank writes its own records and the host merges them by
sample id.
"""
from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass
from typing import List, Optional, Sequence

# B200 roofline denominators used only to ORDER work (LPT); the measured
# peaks in MEASURED_PEAKS.json are what bench.py reports against.
_FP32_FLOPS = 60e12
_HBM_BYTES = 6.4e12
_LAUNCH_S = 4e-6


def predicted_seconds(flops: int, n_bytes: int, launches: int = 6) -> float:
    """Roofline time of one candidate (fwd + grad-input + grad-weights)."""
    return max(3.0 * flops / _FP32_FLOPS, n_bytes / _HBM_BYTES) + launches * _LAUNCH_S


def lpt_shard(costs: Sequence[float], world: int) -> List[List[int]]:
    """Longest-processing-time assignment of candidate indices to ranks.

    Deterministic: candidates are taken by decreasing cost (ties by index)
    and each goes to the least-loaded rank (ties by rank).  Every index
    appears in exactly one shard; shards are returned in index order."""
    if world < 1:
        raise ValueError("world must be >= 1")
    loads = [0.0] * world
    shards: List[List[int]] = [[] for _ in range(world)]
    for i in sorted(range(len(costs)), key=lambda k: (-float(costs[k]), k)):
        r = min(range(world), key=lambda q: (loads[q], q))
        shards[r].append(i)
        loads[r] += float(costs[i])
    return [sorted(s) for s in shards]


@dataclass(frozen=True)
class EvalRecord:
    """One evaluated candidate; ``line()`` follows the reference's sample
    log grammar (search.py:166-171) with the adjoint error as the reward
    field's companion diagnostics."""

    sample_id: int
    seed: int
    flops: int
    params: int
    status: str            # "ok" | "over_budget" | "failed"
    op: str
    seconds: float = 0.0   # device time of fwd + bwd (CUDA events)
    adjoint_err: float = 0.0
    error: str = ""

    def line(self) -> str:
        return (f"sample id={self.sample_id} iter=0 seed={self.seed} reward={0.0!r} flops={self.flops} "
                f"params={self.params} status={self.status} op={self.op}")

    def diag(self) -> str:
        d = f"diag id={self.sample_id} device_us={self.seconds * 1e6:.3f} adjoint_err={self.adjoint_err:.3e}"
        return d + (f" error={self.error}" if self.error else "")


def within_budget(flops: int, params: int, flops_cap: Optional[int], params_cap: Optional[int]) -> bool:
    """pgraph.check_budgets semantics as used by _score_completion (search.py:347-356)."""
    if flops_cap is not None and flops > flops_cap:
        return False
    if params_cap is not None and params > params_cap:
        return False
    return True


def launch(graph, sample_id: int, seed: int, dtype=None, device=None,
           flops_cap: Optional[int] = None, params_cap: Optional[int] = None,
           tol: Optional[float] = None):
    """Enqueue one candidate evaluation on the current CUDA stream without
    waiting for it; returns ``finalize() -> EvalRecord`` (which waits).

    Nothing here synchronises the host with the device: the inner products
    of the adjoint check stay on the device until ``finalize`` reads them,
    so a worker can enqueue the next candidate while this one runs."""
    import torch

    from . import ops
    from .pgraph import handle_for, print_steps

    dtype = dtype or torch.float32
    device = device or torch.device("cuda", torch.cuda.current_device())
    # the rfactored nest (the reference's interpret(staged=True) path, same
    # values): forward runs its stages, backward reverse-mode through them
    h = handle_for(graph, None, True)
    op = print_steps(graph)
    if not within_budget(h.flops_unstaged, h.params, flops_cap, params_cap):
        rec = EvalRecord(sample_id, seed, h.flops_unstaged, h.params, "over_budget", op)
        return lambda: rec
    # one seeded draw for every input (x, the weights, dy), split into views:
    # a candidate is launch-bound, so fewer host-side ops matter
    gen = torch.Generator(device=device).manual_seed(seed)
    shapes = [tuple(h.x_shape)] + [tuple(s) for s in h.w_shapes] + [tuple(h.y_shape)]
    sizes = [math.prod(s) for s in shapes]
    slots = [(n + 7) // 8 * 8 for n in sizes]  # every part starts 16-byte aligned (bf16 and fp32)
    flat = torch.randn(sum(slots), generator=gen, device=device, dtype=torch.float32).to(dtype)
    parts = [p[:n].view(s) for p, n, s in zip(torch.split(flat, slots), sizes, shapes)]
    x, ws, dy = parts[0], parts[1:-1], parts[-1]
    stream = torch.cuda.current_stream(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    try:
        e0.record(stream)
        y = ops.forward(h, x, ws)
        dx, dws = ops.backward(h, x, ws, dy)
        e1.record(stream)
    except Exception as exc:  # a device-engine limit or launch failure: logged like a RewardFailure
        rec = EvalRecord(sample_id, seed, h.flops_unstaged, h.params, "failed", op,
                         error=f"{type(exc).__name__}: {str(exc).splitlines()[0] if str(exc) else ''}"[:200])
        return lambda: rec
    # every inner product in float64 on the device, read once in finalize
    ip = torch.stack([(a.double() * b.double()).sum() for a, b in
                      [(dy, y), (dy, dy), (y, y), (dx, x)] + list(zip(dws, ws))])
    limit = tol if tol is not None else (1e-4 if dtype == torch.float32 else 2e-2 if dtype == torch.bfloat16 else 1e-10)

    def finalize() -> EvalRecord:
        vals = ip.tolist()
        s = vals[0]
        scale = max(1.0, math.sqrt(vals[1] * max(vals[2], 1e-30)))
        err = abs(vals[3] - s) / scale
        for v in vals[4:]:
            err = max(err, abs(v - s) / scale)
        status = "ok" if err <= limit and math.isfinite(err) else "failed"
        return EvalRecord(sample_id, seed, h.flops_unstaged, h.params, status, op, e0.elapsed_time(e1) / 1e3, err)

    return finalize


def evaluate(graph, sample_id: int, seed: int, dtype=None, device=None,
             flops_cap: Optional[int] = None, params_cap: Optional[int] = None,
             tol: Optional[float] = None) -> EvalRecord:
    """Evaluate one candidate on the current CUDA device (and wait for it)."""
    return launch(graph, sample_id, seed, dtype, device, flops_cap, params_cap, tol)()


def candidate_costs(graphs, flops_cap: Optional[int] = None, params_cap: Optional[int] = None) -> List[float]:
    """Predicted seconds per candidate from the native plan (CPU only).

    An over-budget candidate is never executed (``evaluate`` returns before
    any launch, search.py:430-437), so it costs nothing to schedule; pricing
    it by its FLOPs made such phantoms 99% of the predicted total."""
    from .pgraph import handle_for
    out = []
    for g in graphs:
        h = handle_for(g, None, True)
        if not within_budget(h.flops_unstaged, h.params, flops_cap, params_cap):
            out.append(0.0)
            continue
        nbytes = 4 * (2 * math.prod(h.x_shape) + 2 * math.prod(h.y_shape)
                      + 2 * sum(math.prod(s) for s in h.w_shapes))
        out.append(predicted_seconds(h.flops_staged, nbytes))
    return out


def lpt_order(costs: Sequence[float]) -> List[int]:
    """Candidate indices by decreasing predicted cost (ties by index): the
    order a dynamic schedule hands work out in (greedy list scheduling in
    LPT order, within 4/3 of optimal and immune to a cost model that is off
    by a constant factor per class)."""
    return sorted(range(len(costs)), key=lambda k: (-float(costs[k]), k))


class StoreClaim:
    """Dynamic work claiming across ranks through a key-value store's
    atomic counter (torch.distributed's TCPStore: host-side coordination,
    no data-path collective).  ``next()`` returns the next position in the
    shared order, or None when the order is exhausted."""

    def __init__(self, store, n: int, key: str = "syno_sweep_next"):
        self.store, self.n, self.key = store, n, key

    def __call__(self):
        k = int(self.store.add(self.key, 1)) - 1
        return k if k < self.n else None


class LocalClaim:
    """Single-process counterpart of StoreClaim (thread-safe)."""

    def __init__(self, n: int):
        self.n, self.k, self.mu = n, 0, threading.Lock()

    def __call__(self):
        with self.mu:
            if self.k >= self.n:
                return None
            self.k += 1
            return self.k - 1


def claim_loop(order: Sequence[int], claim, work, workers: int = 1) -> list:
    """Run ``work(i)`` for candidates claimed one at a time from ``order``
    by ``workers`` threads until the claim returns None; returns the
    results this process produced (any order)."""
    out, mu = [], threading.Lock()

    def loop():
        while True:
            k = claim()
            if k is None:
                return
            r = work(order[k])
            with mu:
                out.append(r)

    if workers <= 1:
        loop()
        return out
    threads = [threading.Thread(target=loop) for _ in range(workers)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    return out


_TLS = threading.local()


def _worker_stream():
    import torch
    s = getattr(_TLS, "stream", None)
    if s is None:
        s = _TLS.stream = torch.cuda.Stream()
    return s


def _evaluate_on_own_stream(graph, i, seed, dtype, flops_cap, params_cap):
    import torch
    with torch.cuda.stream(_worker_stream()):
        return evaluate(graph, i, seed, dtype=dtype, flops_cap=flops_cap, params_cap=params_cap)


def _launch_on_own_stream(graph, i, seed, dtype, flops_cap, params_cap):
    import torch
    with torch.cuda.stream(_worker_stream()):
        return launch(graph, i, seed, dtype=dtype, flops_cap=flops_cap, params_cap=params_cap)


def run_shard(graphs, indices: Sequence[int], seed0: int = 0, dtype=None, flops_cap=None, params_cap=None,
              workers: int = 1):
    """Evaluate ``graphs[i]`` for i in ``indices`` on this rank's device.

    ``workers > 1`` evaluates that many candidates concurrently, each worker
    thread on its own CUDA stream: most sampled candidates are small
    (launch- and latency-bound), so independent candidates overlap on the
    GPU.  The native library releases the GIL in every call and its
    handles / device plans are safe to use from several threads."""
    t0 = time.perf_counter()
    if workers <= 1:
        recs = [evaluate(graphs[i], i, seed0 + i, dtype=dtype, flops_cap=flops_cap, params_cap=params_cap)
                for i in indices]
        return recs, time.perf_counter() - t0
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=workers) as pool:
        futs = [pool.submit(_evaluate_on_own_stream, graphs[i], i, seed0 + i, dtype, flops_cap, params_cap)
                for i in indices]
        recs = [f.result() for f in futs]
    return recs, time.perf_counter() - t0


def run_dynamic(graphs, order: Sequence[int], claim, seed0: int = 0, dtype=None, flops_cap=None,
                params_cap=None, workers: int = 1):
    """Evaluate candidates claimed dynamically from ``order`` (shared by
    every rank through ``claim``) on this rank's device; each worker thread
    uses its own CUDA stream.  Returns (records, wall seconds)."""
    t0 = time.perf_counter()
    # workers only enqueue (sweep.launch); the records are read once every
    # candidate of this rank is in flight
    pending = claim_loop(order, claim, lambda i: _launch_on_own_stream(graphs[i], i, seed0 + i, dtype, flops_cap,
                                                                       params_cap), workers)
    recs = [f() for f in pending]
    return recs, time.perf_counter() - t0


def merge(shard_records) -> List[EvalRecord]:
    """Host-side merge of per-rank records into one log ordered by sample id."""
    out = [r for recs in shard_records for r in recs]
    out.sort(key=lambda r: r.sample_id)
    ids = [r.sample_id for r in out]
    if len(set(ids)) != len(ids):
        raise ValueError("a candidate was evaluated by two ranks")
    return out

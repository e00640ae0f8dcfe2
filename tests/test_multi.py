"""Multi-process host logic on CPU (gloo, world_size 2): candidate sharding
with no data-path collective, and the proxy-training gradient allreduce.

The device kernels need a GPU; what runs here is everything around them
that decides who evaluates what and how gradients are exchanged.
"""
from __future__ import annotations

import os
import re
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _spawn(fn, world, *args):
    port = _free_port()
    mp.spawn(fn, args=(world, port) + args, nprocs=world, join=True)


def _init(rank, world, port):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


# ---------------------------------------------------------------------------
# LPT sharding
# ---------------------------------------------------------------------------

def test_lpt_partition_and_balance():
    from paper_2410_23745_b200.sweep import lpt_shard
    costs = [float((i * 7919) % 101 + 1) for i in range(257)]
    for world in (1, 2, 3, 4, 8):
        shards = lpt_shard(costs, world)
        flat = sorted(i for s in shards for i in s)
        assert flat == list(range(len(costs)))
        loads = [sum(costs[i] for i in s) for s in shards]
        # LPT bound: max load <= (4/3 - 1/(3m)) OPT <= that times the mean bound
        assert max(loads) <= (4 / 3) * max(sum(costs) / world, max(costs)) + 1e-9
        assert shards == lpt_shard(costs, world)  # deterministic


def test_lpt_edge_cases():
    from paper_2410_23745_b200.sweep import lpt_shard
    assert lpt_shard([], 4) == [[], [], [], []]
    assert lpt_shard([5.0], 3) == [[0], [], []]
    with pytest.raises(ValueError):
        lpt_shard([1.0], 0)
    # equal costs: round-robin by rank
    assert lpt_shard([1.0] * 4, 2) == [[0, 2], [1, 3]]


def test_budget_and_record_line():
    from paper_2410_23745_b200.sweep import EvalRecord, within_budget
    assert within_budget(10, 5, None, None)
    assert not within_budget(11, 5, 10, None)
    assert not within_budget(10, 6, None, 5)
    r = EvalRecord(3, 7, 1000, 64, "ok", "op{reduce(C_in); contract[0:weight,3:both]}", 1e-5, 1e-7)
    # the reference's sample-log grammar (search.py:166-178)
    head, sep, op = r.line().partition(" op=")
    assert sep and op == r.op
    assert re.match(r"^sample id=\d+ iter=\d+ seed=-?\d+ reward=\S+ flops=\d+ params=\d+ status=\w+$", head)


def _sweep_worker(rank, world, port, out_dir):
    _init(rank, world, port)
    from paper_2410_23745_b200 import workloads as WL
    from paper_2410_23745_b200.sweep import candidate_costs, lpt_shard
    graphs = WL.corpus(8, limit=96)
    shards = lpt_shard(candidate_costs(graphs), world)  # every rank computes the same plan
    mine = shards[rank]
    with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
        f.write(" ".join(str(i) for i in mine))
    # the only collective: the barrier the bench uses for timing
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_sweep_shards_cover_corpus_once(tmp_path):
    _spawn(_sweep_worker, 2, str(tmp_path))
    got = []
    for r in range(2):
        txt = (tmp_path / f"rank{r}.txt").read_text().split()
        got.append([int(t) for t in txt])
    assert got[0] and got[1]
    assert sorted(got[0] + got[1]) == list(range(96))


def _claim_worker(rank, world, port, out_dir):
    """The bench's dynamic sweep schedule on gloo: both ranks claim from one
    LPT order through the process group's store; the host merge sees every
    in-budget candidate exactly once."""
    _init(rank, world, port)
    import time as _time

    from paper_2410_23745_b200 import workloads as WL
    from paper_2410_23745_b200.sweep import EvalRecord, StoreClaim, claim_loop, lpt_order, merge
    from paper_2410_23745_b200.sweep import candidate_costs
    graphs = WL.corpus(8, limit=64)
    costs = candidate_costs(graphs, flops_cap=6039797760, params_cap=589824)
    order = lpt_order(costs)
    store = dist.distributed_c10d._get_default_store()
    for step in range(2):
        claim = StoreClaim(store, len(order), f"k{step}")
        dist.barrier()

        def work(i):
            _time.sleep(0.002 * (1 + i % 3))  # stand-in for a device evaluation
            return EvalRecord(i, i, 0, 0, "ok", f"op{i}")
        recs = claim_loop(order, claim, work, workers=3)
        gathered = [None] * world
        dist.all_gather_object(gathered, recs)
        merged = merge(gathered)  # raises on a candidate evaluated twice
        assert [r.sample_id for r in merged] == list(range(len(graphs)))
        assert all(gathered), "both ranks got work"
    if rank == 0:
        with open(os.path.join(out_dir, "ok"), "w") as f:
            f.write("ok")
    dist.destroy_process_group()


def test_gloo_dynamic_claims_cover_corpus_once(tmp_path):
    _spawn(_claim_worker, 2, str(tmp_path))
    assert (tmp_path / "ok").exists()


def test_candidate_costs_ignore_over_budget():
    from paper_2410_23745_b200 import pgraph as P
    from paper_2410_23745_b200 import workloads as WL
    from paper_2410_23745_b200.sweep import candidate_costs, lpt_order, within_budget
    graphs = WL.corpus(8, limit=200)
    fcap, pcap = 6039797760, 589824
    costs = candidate_costs(graphs, fcap, pcap)
    n_over = 0
    for g, c in zip(graphs, costs):
        h = P.handle_for(g, None, True)
        if within_budget(h.flops_unstaged, h.params, fcap, pcap):
            assert c > 0
        else:
            assert c == 0.0
            n_over += 1
    assert n_over > 0
    order = lpt_order(costs)
    assert sorted(order) == list(range(len(graphs)))
    assert all(costs[a] >= costs[b] for a, b in zip(order, order[1:]))


def test_claim_loop_local_threads():
    from paper_2410_23745_b200.sweep import LocalClaim, claim_loop
    order = list(range(50))[::-1]
    got = claim_loop(order, LocalClaim(len(order)), lambda i: i * 2, workers=4)
    assert sorted(got) == [2 * i for i in range(50)]


def test_bench_gpus_mismatch_fails_loudly():
    import subprocess
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)


def test_merge_rejects_duplicates():
    from paper_2410_23745_b200.sweep import EvalRecord, merge
    a = [EvalRecord(0, 0, 1, 1, "ok", "x"), EvalRecord(2, 0, 1, 1, "ok", "x")]
    b = [EvalRecord(1, 0, 1, 1, "ok", "x")]
    assert [r.sample_id for r in merge([a, b])] == [0, 1, 2]
    with pytest.raises(ValueError):
        merge([a, a])


# ---------------------------------------------------------------------------
# Gradient allreduce (proxy training)
# ---------------------------------------------------------------------------

def _grad_worker(rank, world, port, mode):
    _init(rank, world, port)
    from paper_2410_23745_b200.dp import GradBuckets, broadcast_parameters
    torch.manual_seed(100 + rank)  # ranks start different; broadcast fixes that
    model = torch.nn.Sequential(torch.nn.Linear(16, 32), torch.nn.Tanh(), torch.nn.Linear(32, 8))
    broadcast_parameters(list(model.parameters()))
    ref = [p.detach().clone() for p in model.parameters()]
    # tiny buckets so the hook path launches several async allreduces
    buckets = GradBuckets(list(model.parameters()), bucket_bytes=600)
    assert len(buckets.buckets) >= 2
    xs = [torch.randn(4, 16, generator=torch.Generator().manual_seed(r)) for r in range(world)]
    if mode == "hooks":
        buckets.attach()
    out = model(xs[rank]).pow(2).sum()
    out.backward()
    if mode == "hooks":
        buckets.finish()
    else:
        buckets.reduce()
    # expected: the mean over ranks of each rank's gradient, computed locally
    want = [torch.zeros_like(p) for p in ref]
    for r in range(world):
        m2 = torch.nn.Sequential(torch.nn.Linear(16, 32), torch.nn.Tanh(), torch.nn.Linear(32, 8))
        with torch.no_grad():
            for p, q in zip(m2.parameters(), ref):
                p.copy_(q)
        m2(xs[r]).pow(2).sum().backward()
        for w, p in zip(want, m2.parameters()):
            w += p.grad / world
    for p, w in zip(model.parameters(), want):
        assert torch.allclose(p.grad, w, atol=1e-5, rtol=1e-5)
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["sync", "hooks"])
def test_gloo_gradient_allreduce_mean(mode):
    _spawn(_grad_worker, 2, mode)


def _order_worker(rank, world, port):
    """Buckets whose gradients complete out of order (rank 1 produces them in
    reverse) still issue their allreduces in bucket-index order on every rank,
    so the collective sequences match and the means are right."""
    _init(rank, world, port)
    from paper_2410_23745_b200.dp import GradBuckets
    params = [torch.nn.Parameter(torch.zeros(40)) for _ in range(4)]
    gb = GradBuckets(params, bucket_bytes=160).attach()  # one parameter per bucket
    assert len(gb.buckets) == 4
    issued = []
    real = dist.all_reduce

    def spy(t, *a, **k):
        issued.append(next(bi for bi, f in enumerate(gb.flat) if f.data_ptr() == t.data_ptr()))
        return real(t, *a, **k)
    dist.all_reduce = spy
    gb.dist = dist
    seq = params if rank == 0 else params[::-1]
    for k, p in enumerate(seq):
        if rank == 1 and k == 3:
            break  # rank 1 never produces one gradient (an unused parameter)
        p.grad = torch.full_like(p, float(rank + 1))
        gb._stage(p)
    gb.finish()
    dist.all_reduce = real
    assert issued == [0, 1, 2, 3]
    for p in params:
        assert p.grad is not None
    dist.destroy_process_group()


def test_gloo_buckets_issue_in_index_order():
    _spawn(_order_worker, 2)


def test_finish_without_attach_raises():
    from paper_2410_23745_b200.dp import GradBuckets
    lin = torch.nn.Linear(3, 2)
    gb = GradBuckets(list(lin.parameters()))
    with pytest.raises(RuntimeError):
        gb.finish()


def test_grad_buckets_single_process_is_identity():
    from paper_2410_23745_b200.dp import GradBuckets
    lin = torch.nn.Linear(3, 2)
    lin(torch.ones(1, 3)).sum().backward()
    g = [p.grad.clone() for p in lin.parameters()]
    GradBuckets(list(lin.parameters())).reduce()
    for p, w in zip(lin.parameters(), g):
        assert torch.equal(p.grad, w)


def test_bench_sweep_setup_prices_only_executed_candidates():
    """bench.py's cfg5 setup hands the LPT order budget-aware costs: an
    over-budget candidate (never executed, search.py:430-437) costs 0."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2410_23745_b200 import pgraph as P
    from paper_2410_23745_b200.sweep import within_budget
    graphs, costs, fcap, pcap = bench.sweep_setup(limit=120)
    assert len(costs) == len(graphs) == 120
    for g, c in zip(graphs, costs):
        h = P.handle_for(g, None, True)
        assert (c > 0) == within_budget(h.flops_unstaged, h.params, fcap, pcap)


def test_bench_other_configs_are_bench_workloads():
    """The default run's other_configs measure BASELINE's other single-GPU
    configs through the same runners and config descriptions."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    names = [n for n, _ in bench.OTHER_CONFIGS]
    assert names == ["cfg1", "resnet34", "qkv", "sweep"]
    for n, steps in bench.OTHER_CONFIGS:
        assert steps >= 1
        cfg = bench.workload_config(argparse.Namespace(workload=n, batch=0))
        assert cfg["workload"].startswith(("cfg1", "cfg3", "cfg4", "cfg5"))

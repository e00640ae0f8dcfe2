"""Data-parallel proxy training of synthesized operators.

The reference has no trainer (SPEC.md:8 puts it out of scope); the paper's
proxy training replaces GPT-2's QKV projections with synthesized operators
(PAPER.md:619).  This module is the B200 equivalent: one process per GPU,
each rank runs forward + backward of its own batch through the device
kernels (ops.SynoFunction), and the weight gradients are averaged with
ONE exchange step -- an allreduce over NVLink/NVSwitch through
torch.distributed's NCCL backend (gloo in the CPU tests).  Gradients are
packed into flat buckets so the collective count per step is small and
fixed, and each bucket's allreduce is launched asynchronously as soon as
the bucket's last gradient is produced, overlapping communication with the
rest of the backward pass.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch


class GradBuckets:
    """Flat gradient buckets with async allreduce (mean over ranks).

    Parameters are bucketed in REVERSE registration order (the order the
    backward pass produces their gradients), ``bucket_bytes`` per bucket.
    ``attach()`` registers post-accumulate hooks that copy each gradient
    into its bucket and fire the bucket's allreduce once complete;
    ``finish()`` waits and writes the averaged values back to ``.grad``.
    Without ``attach()``, ``reduce()`` does the same synchronously.
    """

    def __init__(self, params: Sequence[torch.nn.Parameter], bucket_bytes: int = 32 << 20, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.params = [p for p in params if p.requires_grad]
        self.buckets: List[List[torch.nn.Parameter]] = []
        cur, size = [], 0
        for p in reversed(self.params):
            nb = p.numel() * p.element_size()
            if cur and (size + nb > bucket_bytes or p.dtype != cur[0].dtype or p.device != cur[0].device):
                self.buckets.append(cur)
                cur, size = [], 0
            cur.append(p)
            size += nb
        if cur:
            self.buckets.append(cur)
        self.flat = [torch.empty(sum(p.numel() for p in b), dtype=b[0].dtype, device=b[0].device)
                     for b in self.buckets]
        self.where = {}
        for bi, b in enumerate(self.buckets):
            off = 0
            for p in b:
                self.where[id(p)] = (bi, off)
                off += p.numel()
        self.pending = [0] * len(self.buckets)
        self.works: List[Optional[object]] = [None] * len(self.buckets)
        self.hooks = []
        # collectives are issued strictly in bucket-index order on every rank
        # (a bucket that completes early waits for its predecessors), so the
        # NCCL call sequence cannot diverge across ranks
        self.next_launch = 0

    def _stage(self, p):
        bi, off = self.where[id(p)]
        self.flat[bi][off:off + p.numel()].copy_(p.grad.reshape(-1))
        self.pending[bi] += 1
        self._launch_ready()

    def _launch_ready(self):
        while self.next_launch < len(self.buckets) and \
                self.pending[self.next_launch] == len(self.buckets[self.next_launch]):
            bi = self.next_launch
            if self.world > 1:
                self.works[bi] = self.dist.all_reduce(self.flat[bi], op=self.dist.ReduceOp.SUM, group=self.group,
                                                      async_op=True)
            self.next_launch += 1

    def attach(self):
        for p in self.params:
            self.hooks.append(p.register_post_accumulate_grad_hook(self._stage))
        return self

    def detach(self):
        for h in self.hooks:
            h.remove()
        self.hooks = []

    def finish(self):
        if not self.hooks and any(self.pending[bi] != len(b) for bi, b in enumerate(self.buckets)):
            raise RuntimeError("GradBuckets.finish() without attach(): call reduce() for the synchronous path")
        # unused parameters contribute zeros; their buckets then launch in index order
        for bi, b in enumerate(self.buckets):
            if self.pending[bi] != len(b):
                for p in b:
                    if p.grad is None:
                        p.grad = torch.zeros_like(p)
                        self._stage(p)
        assert self.next_launch == len(self.buckets)
        for bi, b in enumerate(self.buckets):
            w = self.works[bi]
            if w is not None:
                w.wait()
            if self.world > 1:
                self.flat[bi].div_(self.world)
            off = 0
            for p in b:
                p.grad.copy_(self.flat[bi][off:off + p.numel()].view_as(p.grad))
                off += p.numel()
            self.pending[bi] = 0
            self.works[bi] = None
        self.next_launch = 0

    def reduce(self):
        """Synchronous path: stage every gradient, allreduce, write back."""
        for p in self.params:
            if p.grad is None:
                p.grad = torch.zeros_like(p)
        self.next_launch = 0
        for bi, b in enumerate(self.buckets):
            self.pending[bi] = 0
        for bi, b in enumerate(self.buckets):
            for p in b:
                self._stage(p)
        self.finish()


def broadcast_parameters(params: Sequence[torch.nn.Parameter], src: int = 0, group=None):
    """Make every rank start from rank ``src``'s weights."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    with torch.no_grad():
        for p in params:
            dist.broadcast(p.data, src=src, group=group)


class ProxyQKV(torch.nn.Module):
    """GPT-2-small-shaped proxy: ``layers`` QKV projections, each a
    synthesized operator over (T, E) -> (T, E3), with a tanh between them
    projected back to E by slicing (keeps every layer's input shape)."""

    def __init__(self, graph, layers: int = 12, dtype=torch.bfloat16, device=None, seed: int = 0):
        super().__init__()
        from .ops import SynoOperator
        self.ops = torch.nn.ModuleList(
            [SynoOperator(graph, dtype=dtype, device=device, seed=seed + k) for k in range(layers)])

    def forward(self, x):
        e = x.shape[-1]
        for op in self.ops:
            x = torch.tanh(op(x)[..., :e])
        return x


def train_step(model, buckets: GradBuckets, x, target, lr: float = 1e-3):
    """One proxy-training step: fwd, bwd (device kernels), bucketed allreduce, SGD."""
    for p in buckets.params:
        p.grad = None
    out = model(x)
    loss = torch.nn.functional.mse_loss(out.float(), target.float())
    loss.backward()
    buckets.finish()
    with torch.no_grad():
        for p in buckets.params:
            p.add_(p.grad, alpha=-lr)
    return loss.detach()

"""Device-resident fit reward (reference reward.py).

The reference scores a candidate by fitting its weights to imitate a
target operator: per weight tensor, a matrix-free least-squares solve with
``scipy.sparse.linalg.lsqr`` whose matvec is ``interpret`` and whose
rmatvec is ``weight_gradient`` (reward.py:99-131), alternating over
tensors (reward.py:134-172); reward = exp(-residual / target energy).

Here the same algorithm runs with every vector on the GPU in float64: the
matvec / rmatvec are the backend's forward and weight-gradient kernels on
device tensors, and LSQR (Paige & Saunders; the recurrences and stopping
rules of scipy's ``lsqr``, restated in ``lsqr_device``) keeps its
iterates in HBM.  Only scalar norms cross to the host, to evaluate the
stopping tests.  Names and argument meaning follow the reference:

    fit_target(spec, op_text, seed=0, samples=2, assignment=None)      reward.py:72-92
    builtin_fit_reward(graph, target, seed=0, sweeps=2, assignment=None)  reward.py:134-172
    make_reward_fn(backend)                                             reward.py:229-246
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Mapping, Optional

import numpy as np

from .codegen import input_shape, random_weights, weight_shapes
from .pgraph import handle_for, parse_steps, print_steps

_EPS = float(np.finfo(np.float64).eps)


@dataclass(frozen=True)
class RewardReport:
    reward: float
    diagnostics: tuple = ()

    def diag(self, key: str) -> Optional[str]:
        for k, v in self.diagnostics:
            if k == key:
                return v
        return None


def _clip(value: float) -> float:
    if not math.isfinite(value):
        return 0.0
    return min(1.0, max(0.0, value))


@dataclass(frozen=True, eq=False)
class FitTarget:
    """Seeded regression problem; ``xs``/``ys`` are float64 CUDA tensors."""

    xs: tuple
    ys: tuple
    norm: float
    label: str


def fit_target(spec, op_text: str, seed: int = 0, samples: int = 2,
               assignment: Optional[Mapping[str, int]] = None) -> FitTarget:
    """reward.fit_target: the same numpy draws (weights, then inputs) as the
    reference, so the regression problem is identical; evaluated on the GPU."""
    import torch

    from . import ops
    target = parse_steps(op_text, spec)
    rng = np.random.default_rng(seed)
    tw = random_weights(target, rng, assignment)
    shape = input_shape(spec, assignment)
    xs_np = [rng.standard_normal(shape) for _ in range(samples)]
    h = handle_for(target, assignment)
    twd = [ops.to_device(w, "float64") for w in tw]
    xs = tuple(ops.to_device(x, "float64") for x in xs_np)
    ys = tuple(ops.forward(h, x, twd) for x in xs)
    norm = float(sum(float(torch.sum(y * y)) for y in ys))
    return FitTarget(xs=xs, ys=ys, norm=norm, label=op_text)


def _sym_ortho(a: float, b: float):
    """Stable Givens rotation (c, s, r) with r = hypot(a, b)."""
    if b == 0:
        return math.copysign(1.0, a) if a != 0 else 0.0, 0.0, abs(a)
    if a == 0:
        return 0.0, math.copysign(1.0, b), abs(b)
    if abs(b) > abs(a):
        tau = a / b
        s = math.copysign(1.0, b) / math.sqrt(1 + tau * tau)
        return s * tau, s, b / s
    tau = b / a
    c = math.copysign(1.0, a) / math.sqrt(1 + tau * tau)
    return c, c * tau, a / c


def lsqr_device(matvec, rmatvec, b, n: int, atol: float = 1e-10, btol: float = 1e-10,
                conlim: float = 1e8, iter_lim: Optional[int] = None):
    """LSQR (damp = 0) on device vectors; returns (x, istop, itn)."""
    import torch
    iter_lim = iter_lim if iter_lim is not None else 2 * n
    x = torch.zeros(n, dtype=torch.float64, device=b.device)
    u = b.clone()
    bnorm = float(torch.linalg.vector_norm(b))
    beta = bnorm
    if beta > 0:
        u = u / beta
        v = rmatvec(u)
        alfa = float(torch.linalg.vector_norm(v))
    else:
        v = torch.zeros_like(x)
        alfa = 0.0
    if alfa > 0:
        v = v / alfa
    w = v.clone()
    rhobar, phibar = alfa, beta
    anorm = acond = ddnorm = res2 = xnorm = xxnorm = z = 0.0
    cs2, sn2 = -1.0, 0.0
    ctol = 1.0 / conlim if conlim > 0 else 0.0
    if alfa * beta == 0:
        return x, 0, 0
    itn, istop = 0, 0
    while itn < iter_lim:
        itn += 1
        u = matvec(v) - alfa * u
        beta = float(torch.linalg.vector_norm(u))
        if beta > 0:
            u = u / beta
            anorm = math.sqrt(anorm * anorm + alfa * alfa + beta * beta)
            v = rmatvec(u) - beta * v
            alfa = float(torch.linalg.vector_norm(v))
            if alfa > 0:
                v = v / alfa
        cs, sn, rho = _sym_ortho(rhobar, beta)
        theta = sn * alfa
        rhobar = -cs * alfa
        phi = cs * phibar
        phibar = sn * phibar
        tau = sn * phi
        t1, t2 = phi / rho, -theta / rho
        dk = w / rho
        x = x + t1 * w
        w = v + t2 * w
        ddnorm += float(torch.sum(dk * dk))
        delta = sn2 * rho
        gambar = -cs2 * rho
        rhs = phi - delta * z
        zbar = rhs / gambar
        xnorm = math.sqrt(xxnorm + zbar * zbar)
        gamma = math.sqrt(gambar * gambar + theta * theta)
        cs2, sn2 = gambar / gamma, theta / gamma
        z = rhs / gamma
        xxnorm += z * z
        acond = anorm * math.sqrt(ddnorm)
        rnorm = math.sqrt(phibar * phibar + res2)
        arnorm = alfa * abs(tau)
        test1 = rnorm / bnorm
        test2 = arnorm / (anorm * rnorm + _EPS)
        test3 = 1.0 / (acond + _EPS)
        t1 = test1 / (1 + anorm * xnorm / bnorm)
        rtol = btol + atol * anorm * xnorm / bnorm
        if itn >= iter_lim:
            istop = 7
        if 1 + test3 <= 1:
            istop = 6
        if 1 + test2 <= 1:
            istop = 5
        if 1 + t1 <= 1:
            istop = 4
        if test3 <= ctol:
            istop = 3
        if test2 <= atol:
            istop = 2
        if test1 <= rtol:
            istop = 1
        if istop:
            break
    return x, istop, itn


def _solve_weight(h, target: FitTarget, weights: list, index: int) -> list:
    """reward._solve_weight (reward.py:99-131) with device matvec / rmatvec."""
    import torch

    from . import ops
    shape = tuple(weights[index].shape)
    n = int(np.prod(shape)) if shape else 1
    sizes = [y.numel() for y in target.ys]

    def matvec(vec):
        trial = list(weights)
        trial[index] = vec.reshape(shape)
        return torch.cat([ops.forward(h, x, trial).reshape(-1) for x in target.xs])

    def rmatvec(u):
        grad = torch.zeros(n, dtype=torch.float64, device=u.device)
        off = 0
        for x, y, m in zip(target.xs, target.ys, sizes):
            piece = u[off:off + m].reshape(y.shape)
            off += m
            want = [j == index for j in range(len(weights))]
            _, dws = ops.backward(h, x, weights, piece, want_dx=False, want_dw=want)
            grad += dws[index].reshape(-1)
        return grad

    rhs = torch.cat([y.reshape(-1) for y in target.ys])
    sol, _, _ = lsqr_device(matvec, rmatvec, rhs, n, atol=1e-10, btol=1e-10, iter_lim=max(2 * n, 40))
    out = list(weights)
    out[index] = sol.reshape(shape)
    return out


def builtin_fit_reward(graph, target: FitTarget, seed: int = 0, sweeps: int = 2,
                       assignment: Optional[Mapping[str, int]] = None) -> RewardReport:
    """reward.builtin_fit_reward (reward.py:134-172), iterates on the GPU."""
    import torch

    from . import ops
    h = handle_for(graph, assignment)
    shapes = weight_shapes(graph, assignment)
    weights = []
    if shapes:
        weights = [ops.to_device(w, "float64")
                   for w in random_weights(graph, np.random.default_rng(seed + 1), assignment)]
        for _ in range(sweeps if len(shapes) > 1 else 1):
            for index in range(len(shapes)):
                weights = _solve_weight(h, target, weights, index)
    residual = float(sum(float(torch.sum((ops.forward(h, x, weights) - y) ** 2))
                         for x, y in zip(target.xs, target.ys)))
    if not math.isfinite(residual):
        return RewardReport(0.0, (("error", "singular fit"),))
    norm = target.norm if target.norm > 0 else 1.0
    return RewardReport(_clip(math.exp(-residual / norm)),
                        (("residual", repr(residual)), ("target_norm", repr(target.norm)),
                         ("weights", str(len(shapes)))))


def make_reward_fn(backend: Callable) -> Callable:
    """reward.make_reward_fn (reward.py:229-246): memoised by serialized steps."""
    memo: dict = {}

    def reward_fn(graph) -> float:
        key = print_steps(graph)
        hit = memo.get(key)
        if hit is None:
            hit = backend(graph).reward
            memo[key] = hit
        return hit

    return reward_fn

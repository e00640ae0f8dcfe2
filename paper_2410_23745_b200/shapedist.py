"""Shape-distance mirror (reference: opsmith/shapedist.py) on the native solver.

The search estimates "at least how many more steps until the frontier can
match the input?" by partitioning the frontier and the input dims into
reshape groups (shapedist.py:1-40).  The reference runs that memoised
partition search in Python, where it is ~73% of MCTS CPU time (SURVEY §2,
§8(f)4); here it runs in ``csrc/shapedist.cpp`` behind
``syno_shape_distance`` / ``syno_graph_distance`` (include/syno.h).

Names, arguments and results follow the reference:

    shape_distance(current, input_dims, may_reduce=False) -> float   (shapedist.py:405-412)
    explain_distance(current, input_dims, may_reduce=False)          (shapedist.py:377-402)
    graph_distance(graph) -> float                                   (shapedist.py:415-420)
    group_cost(ReshapeGroup) -> int                                  (shapedist.py:76-87)

``current`` holds ``DimDesc`` objects or bare sizes; a size is the
reference's ``SymbolicSize`` (anything with ``.powers``) or its text form
("H*s^-1", "K^2", "1").  ``explain_distance`` returns one optimal grouping;
when several are optimal it may differ from the reference's (whose choice
depends on its interning history), the distance never does.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

from . import _lib
from .errors import raise_status

INF = float("inf")


@dataclass(frozen=True)
class DimDesc:
    """What the distance needs to know about one frontier dim (shapedist.py:55-61)."""

    size: object
    reduce_pure: bool = False
    strided: bool = False


def desc_of_dim(d) -> DimDesc:
    return DimDesc(d.size, d.reduce_pure, d.strided)


def _powers(size) -> tuple:
    """((variable name, exponent), ...) of a size, zero exponents dropped."""
    if isinstance(size, DimDesc):
        size = size.size
    pw = getattr(size, "powers", None)
    acc: dict = {}
    if pw is not None:
        for v, e in pw:
            name = getattr(v, "name", v)
            acc[name] = acc.get(name, 0) + int(e)
    else:
        text = str(size).replace(" ", "")
        if text and text != "1":
            for factor in text.split("*"):
                name, _, exp = factor.partition("^")
                if not name:
                    raise ValueError(f"bad size text {size!r}")
                acc[name] = acc.get(name, 0) + (int(exp) if exp else 1)
    return tuple(sorted((n, e) for n, e in acc.items() if e))


@dataclass(frozen=True)
class ReshapeGroup:
    lhs: tuple
    rhs: tuple

    @property
    def needs_elimination(self) -> bool:
        return _total(self.lhs) != _total(self.rhs)


def _total(sizes) -> tuple:
    acc: dict = {}
    for s in sizes:
        for n, e in _powers(s):
            acc[n] = acc.get(n, 0) + e
    return tuple(sorted((n, e) for n, e in acc.items() if e))


def group_cost(group: ReshapeGroup) -> int:
    """Balanced groups cost |lhs| + |rhs| - 2; eliminating ones one more, at least 1 (shapedist.py:76-87)."""
    n = len(group.lhs) + len(group.rhs)
    if group.needs_elimination:
        return max(n - 1, 1)
    return max(n - 2, 0)


@dataclass(frozen=True)
class DistanceResult:
    distance: float
    groups: tuple = ()
    permutation: Optional[tuple] = None


def _encode(descs: Sequence[DimDesc], inputs: Sequence) -> tuple:
    var_ids: dict = {}

    def terms(size):
        out = []
        for name, e in _powers(size):
            out += [var_ids.setdefault(name, len(var_ids)), e]
        return out

    d_n, d_t, flags = [], [], []
    for d in descs:
        t = terms(d.size)
        d_n.append(len(t) // 2)
        d_t += t
        flags.append((1 if d.reduce_pure else 0) | (2 if d.strided else 0))
    i_n, i_t = [], []
    for s in inputs:
        t = terms(s)
        i_n.append(len(t) // 2)
        i_t += t
    I32 = ctypes.c_int32
    return ((I32 * max(len(d_n), 1))(*d_n), (I32 * max(len(d_t), 1))(*d_t),
            (ctypes.c_uint8 * max(len(flags), 1))(*flags), (I32 * max(len(i_n), 1))(*i_n),
            (I32 * max(len(i_t), 1))(*i_t))


def _as_descs(current) -> list:
    return [d if isinstance(d, DimDesc) else DimDesc(d) for d in current]


def _solve(current, input_dims, may_reduce: bool, groups: bool):
    descs = _as_descs(current)
    inputs = list(input_dims)
    d_n, d_t, flags, i_n, i_t = _encode(descs, inputs)
    out = ctypes.c_double(0.0)
    dg = (ctypes.c_int32 * max(len(descs), 1))() if groups else None
    ig = (ctypes.c_int32 * max(len(inputs), 1))() if groups else None
    ng = ctypes.c_int32(0)
    rc = _lib.lib.syno_shape_distance(len(descs), d_n, d_t, flags, len(inputs), i_n, i_t, int(bool(may_reduce)),
                                      ctypes.byref(out), dg, ig, ctypes.byref(ng) if groups else None)
    if rc:
        raise_status(rc, _lib.last_error())
    return descs, inputs, out.value, dg, ig, ng.value


def shape_distance(current: Sequence, input_dims: Sequence, may_reduce: bool = False) -> float:
    """shapedist.shape_distance (shapedist.py:405-412)."""
    return _solve(current, input_dims, may_reduce, False)[2]


def explain_distance(current: Sequence, input_dims: Sequence, may_reduce: bool = False) -> DistanceResult:
    """shapedist.explain_distance (shapedist.py:377-402): distance, one optimal
    grouping and, at distance 0, the frontier-to-input permutation."""
    descs, inputs, dist, dg, ig, ng = _solve(current, input_dims, may_reduce, True)
    if dist == INF:
        return DistanceResult(INF)
    groups = tuple(
        ReshapeGroup(tuple(d.size for k, d in enumerate(descs) if dg[k] == g),
                     tuple(s for k, s in enumerate(inputs) if ig[k] == g))
        for g in range(ng))
    perm = None
    if dist == 0:
        used: set = set()
        order = []
        for size in inputs:
            want = _powers(size)
            for k, d in enumerate(descs):
                if k not in used and _powers(d.size) == want:
                    used.add(k)
                    order.append(k)
                    break
        perm = tuple(order)
    return DistanceResult(dist, groups, perm)


def graph_distance(graph) -> float:
    """shapedist.graph_distance (shapedist.py:415-420) of one of our PGraphs
    (replayed natively) or of a reference PGraph (its frontier dims)."""
    from .pgraph import Handle, PGraph, operator_document

    if isinstance(graph, PGraph) or not hasattr(graph, "dims"):
        h = Handle(operator_document(graph), None, False, replay_only=True)
        out = ctypes.c_double(0.0)
        rc = _lib.lib.syno_graph_distance(h.ptr, ctypes.byref(out))
        if rc:
            raise_status(rc, _lib.last_error())
        return out.value
    return shape_distance([desc_of_dim(d) for d in graph.dims], graph.spec.input_dims,
                          may_reduce=graph.in_reduction)


def clear_cache() -> None:
    """shapedist.clear_cache (shapedist.py:423-433)."""
    _lib.lib.syno_shape_distance_clear_cache()

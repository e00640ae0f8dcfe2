"""Execution API mirror (reference: opsmith/codegen.py), running on the B200.

Same names, argument meaning and error behaviour as the reference:

    interpret(graph, x, weights=(), assignment=None, staged=False)     codegen.py:598-630
    weight_gradient(graph, x, upstream, weights, assignment=None)      codegen.py:664-743
    flops(graph, assignment=None, staged=False)                        codegen.py:633-651
    param_count(graph, assignment=None)                                codegen.py:654-657
    input_shape / output_shape / weight_shapes / random_weights        codegen.py:575-595
    emit_loop_nest / parse_loop_nest / run_nest                        codegen.py:750-794, 846-943, 549-572

plus ``input_gradient`` (the adjoint of the x access),
which the reference does not have.

numpy arguments are computed in float64 on the GPU and returned as numpy
float64 arrays, so the reference's own callers (e.g. reward.builtin_fit_reward's
lsqr) see the precision they expect.  torch CUDA tensors are computed in
their own dtype (float32 / bfloat16 / float64) and returned as torch tensors.
Nothing here computes on the CPU: without a CUDA device these raise.
"""
from __future__ import annotations

from typing import Mapping, Optional, Sequence

import numpy as np

from .errors import LoopNestParseError, OperatorParseError, ShapeMismatch
from .pgraph import Handle, PGraph, handle_for, operator_document, spec_header

__all__ = [
    "ShapeMismatch", "interpret", "weight_gradient", "input_gradient", "flops", "param_count",
    "input_shape", "output_shape", "weight_shapes", "random_weights", "emit_loop_nest",
    "LoopNest", "LoopNestParseError", "parse_loop_nest", "run_nest",
]


def _spec_name(graph) -> str:
    return graph.spec.name


def input_shape(spec, assignment: Optional[Mapping[str, int]] = None) -> tuple:
    from .pgraph import ProblemSpec  # noqa: F401  (spec may be ours or the reference's)
    env = dict(assignment) if assignment is not None else dict(spec.reference)
    from ._sizes import eval_size_text
    return tuple(eval_size_text(str(s), env) for s in tuple(spec.batch_dims) + tuple(spec.input_dims))


def output_shape(spec, assignment: Optional[Mapping[str, int]] = None) -> tuple:
    env = dict(assignment) if assignment is not None else dict(spec.reference)
    from ._sizes import eval_size_text
    return tuple(eval_size_text(str(s), env) for s in tuple(spec.batch_dims) + tuple(spec.output_dims))


def weight_shapes(graph, assignment: Optional[Mapping[str, int]] = None) -> list:
    return [tuple(s) for s in handle_for(graph, assignment).w_shapes]


def random_weights(graph, rng: np.random.Generator, assignment: Optional[Mapping[str, int]] = None) -> list:
    """codegen.random_weights (codegen.py:590-595): N(0,1) draws in weight order."""
    return [rng.standard_normal(shape) for shape in weight_shapes(graph, assignment)]


def flops(graph, assignment: Optional[Mapping[str, int]] = None, staged: bool = False) -> int:
    h = handle_for(graph, assignment)
    return int(h.flops_staged if staged else h.flops_unstaged)


def param_count(graph, assignment: Optional[Mapping[str, int]] = None) -> int:
    return int(handle_for(graph, assignment).params)


def emit_loop_nest(graph, assignment: Optional[Mapping[str, int]] = None, staged: bool = False) -> str:
    """codegen.emit_loop_nest(build_loop_nest(graph)) or of its rfactor staging;
    of a parsed ``LoopNest``, its own text (the reference's round trip)."""
    if isinstance(graph, LoopNest):
        return graph.handle.emit(False)
    return handle_for(graph, assignment).emit(staged)


class LoopNest:
    """A loop nest parsed from text (codegen.LoopNest via parse_loop_nest), held
    by the native library as an executable handle (``syno_compile_nest``)."""

    def __init__(self, handle: Handle, assignment: tuple):
        self.handle = handle
        self.assignment = assignment

    @property
    def name(self) -> str:
        return self.text.splitlines()[0][len("nest "):]

    @property
    def text(self) -> str:
        return self.handle.emit(False)

    @property
    def n_stages(self) -> int:
        return int(self.handle.info.n_forward_stages)

    def __eq__(self, other) -> bool:
        return isinstance(other, LoopNest) and (self.text, self.assignment) == (other.text, other.assignment)

    def __hash__(self):
        return hash((self.text, self.assignment))


def parse_loop_nest(text: str, spec, assignment: Optional[Mapping[str, int]] = None) -> LoopNest:
    """codegen.parse_loop_nest (codegen.py:846-943): the inverse of
    emit_loop_nest under a spec's variables (ours or the reference's);
    extents from the spec's reference assignment unless one is given.
    Raises LoopNestParseError for malformed text."""
    try:
        h = Handle(spec_header(spec), assignment, False, nest_text=text)
    except OperatorParseError as exc:
        raise LoopNestParseError(str(exc)) from None
    env = dict(assignment) if assignment is not None else dict(spec.reference)
    return LoopNest(h, tuple(sorted((k, int(v)) for k, v in env.items())))


def run_nest(nest: LoopNest, x, weights: Sequence = ()):
    """codegen.run_nest (codegen.py:549-572): one element (no batch axes)
    through a parsed nest's stages on the GPU.  numpy in -> float64 -> numpy
    out; torch CUDA tensors in their own dtype."""
    from . import ops
    h = nest.handle
    torch_in = _is_torch(x)
    if not torch_in:
        x = np.asarray(x, dtype=np.float64)
        weights = [np.asarray(w, dtype=np.float64) for w in weights]
    if len(weights) != h.n_weights:
        raise ShapeMismatch(f"{nest.name}: expected {h.n_weights} weight tensors, got {len(weights)}")
    if tuple(x.shape) != h.x_shape:
        raise ShapeMismatch(f"{nest.name}: expected input shape {h.x_shape}, got {tuple(x.shape)}")
    for j, (w, want) in enumerate(zip(weights, h.w_shapes)):
        if tuple(w.shape) != tuple(want):
            raise ShapeMismatch(f"w{j}: expected shape {tuple(want)}, got {tuple(w.shape)}")
    if torch_in:
        return ops.forward(h, x, list(weights))
    xd, *wd = _to_device([x] + list(weights), "float64")
    return ops.to_numpy(ops.forward(h, xd, wd))


# ---------------------------------------------------------------------------
# Device execution
# ---------------------------------------------------------------------------

def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _check_common(graph, h, x_shape, weights):
    if len(weights) != h.n_weights:
        raise ShapeMismatch(f"{_spec_name(graph)}: expected {h.n_weights} weight tensors, got {len(weights)}")
    if tuple(x_shape) != h.x_shape:
        raise ShapeMismatch(f"{_spec_name(graph)}: expected input shape {h.x_shape}, got {tuple(x_shape)}")
    for j, (w, want) in enumerate(zip(weights, h.w_shapes)):
        if tuple(w.shape) != tuple(want):
            raise ShapeMismatch(f"w{j}: expected shape {tuple(want)}, got {tuple(w.shape)}")


def _to_device(arrays, dtype):
    from . import ops
    return [ops.to_device(a, dtype) for a in arrays]


def interpret(graph, x, weights: Sequence = (), assignment: Optional[Mapping[str, int]] = None,
              staged: bool = False):
    """Run an operator on an input tensor (leading batch axes allowed)."""
    from . import ops
    h = handle_for(graph, assignment, staged)
    torch_in = _is_torch(x)
    if not torch_in:
        x = np.asarray(x, dtype=np.float64)
        weights = [np.asarray(w, dtype=np.float64) for w in weights]
    _check_common(graph, h, x.shape, list(weights))
    if torch_in:
        return ops.forward(h, x, list(weights))
    xd, *wd = _to_device([x] + list(weights), "float64")
    return ops.to_numpy(ops.forward(h, xd, wd))


def _grads(graph, x, upstream, weights, assignment, want_dx, want_dw):
    from . import ops
    h = handle_for(graph, assignment)
    torch_in = _is_torch(x)
    if not torch_in:
        x = np.asarray(x, dtype=np.float64)
        upstream = np.asarray(upstream, dtype=np.float64)
        weights = [np.asarray(w, dtype=np.float64) for w in weights]
    if tuple(x.shape) != h.x_shape:
        raise ShapeMismatch(f"expected input shape {h.x_shape}, got {tuple(x.shape)}")
    if tuple(upstream.shape) != h.y_shape:
        raise ShapeMismatch(f"expected upstream shape {h.y_shape}, got {tuple(upstream.shape)}")
    if len(weights) != h.n_weights:
        raise ShapeMismatch(f"expected {h.n_weights} weight tensors, got {len(weights)}")
    _check_common(graph, h, x.shape, list(weights))
    if torch_in:
        return ops.backward(h, x, list(weights), upstream, want_dx, want_dw)
    xd, ud, *wd = _to_device([x, upstream] + list(weights), "float64")
    dx, dws = ops.backward(h, xd, wd, ud, want_dx, want_dw)
    return (ops.to_numpy(dx) if dx is not None else None), [ops.to_numpy(g) if g is not None else None for g in dws]


def weight_gradient(graph, x, upstream, weights: Sequence, assignment: Optional[Mapping[str, int]] = None) -> list:
    """Gradient of <upstream, output> with respect to each weight."""
    return _grads(graph, x, upstream, weights, assignment, False, True)[1]


def input_gradient(graph, x, upstream, weights: Sequence = (), assignment: Optional[Mapping[str, int]] = None):
    """Gradient of <upstream, output> with respect to the input x."""
    return _grads(graph, x, upstream, weights, assignment, True, False)[0]


def gradients(graph, x, upstream, weights: Sequence = (), assignment: Optional[Mapping[str, int]] = None):
    """(dX, [dW_j]) in one call."""
    return _grads(graph, x, upstream, weights, assignment, True, True)


# ---------------------------------------------------------------------------
# Tensor file format (codegen.save_tensor / load_tensor, codegen.py:950-976),
# implemented by the native library (syno_tensor_write / syno_tensor_read)
# ---------------------------------------------------------------------------

def save_tensor(path, array) -> None:
    """rank, then dims, as little-endian int64; float64 row-major payload."""
    import ctypes

    from . import _lib
    from .errors import raise_status
    arr = np.array(array, dtype="<f8", order="C", copy=True)  # keeps 0-d arrays 0-d
    dims = (ctypes.c_int64 * max(1, arr.ndim))(*arr.shape)
    rc = _lib.lib.syno_tensor_write(str(path).encode(), arr.ndim, dims,
                                    arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if rc:
        raise_status(rc, _lib.last_error())


def load_tensor(path) -> np.ndarray:
    import ctypes

    from . import _lib
    from .errors import raise_status
    rank, count = ctypes.c_int(0), ctypes.c_int64(0)
    dims = (ctypes.c_int64 * _lib.MAX_RANK)()
    rc = _lib.lib.syno_tensor_read(str(path).encode(), ctypes.byref(rank), dims, None, 0, ctypes.byref(count))
    if rc:
        raise_status(rc, _lib.last_error())
    out = np.empty(tuple(dims[k] for k in range(rank.value)), dtype="<f8")
    rc = _lib.lib.syno_tensor_read(str(path).encode(), ctypes.byref(rank), dims,
                                   out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), out.size,
                                   ctypes.byref(count))
    if rc:
        raise_status(rc, _lib.last_error())
    return out


__all__ += ["gradients", "PGraph", "operator_document", "save_tensor", "load_tensor"]

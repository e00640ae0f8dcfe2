"""torch integration: device buffers, streams, autograd.

torch is plumbing here (allocation, the current CUDA stream, autograd
bookkeeping); every arithmetic operation happens inside libsyno.so kernels
launched through the C ABI on torch's current stream.
"""
from __future__ import annotations

import ctypes
from typing import Mapping, Optional, Sequence

import numpy as np
import torch

from . import _lib
from .errors import raise_status
from .pgraph import Handle, handle_for

_DT = {torch.float32: _lib.SYNO_F32, torch.bfloat16: _lib.SYNO_BF16, torch.float64: _lib.SYNO_F64}
_NAMES = {"float32": torch.float32, "bfloat16": torch.bfloat16, "float64": torch.float64}


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("the syno B200 backend needs a CUDA device; there is no CPU fallback")


def to_device(a, dtype: str = "float64", device: Optional[torch.device] = None) -> torch.Tensor:
    require_cuda()
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
    return t.to(device=device or torch.device("cuda"), dtype=_NAMES[dtype]).contiguous()


def to_numpy(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").numpy()


def _ptr(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream_ptr(t: torch.Tensor):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _code(tensors) -> int:
    dts = {t.dtype for t in tensors}
    if len(dts) != 1:
        raise TypeError(f"operator tensors must share one dtype, got {sorted(str(d) for d in dts)}")
    dt = dts.pop()
    if dt not in _DT:
        raise TypeError(f"unsupported dtype {dt}")
    for t in tensors:
        if not t.is_cuda:
            raise ValueError("operator tensors must be CUDA tensors")
    return _DT[dt]


def forward(h: Handle, x: torch.Tensor, weights: Sequence[torch.Tensor], out: Optional[torch.Tensor] = None):
    x = x.contiguous()
    weights = [w.contiguous() for w in weights]
    code = _code([x] + weights)
    y = out if out is not None else torch.empty(h.y_shape, dtype=x.dtype, device=x.device)
    warr = (ctypes.c_void_p * max(1, len(weights)))(*[w.data_ptr() for w in weights])
    with torch.cuda.device(x.device):
        rc = _lib.lib.syno_forward(h.ptr, code, _ptr(x), warr, len(weights), _ptr(y), _stream_ptr(x))
    if rc:
        raise_status(rc, _lib.last_error())
    return y


def backward(h: Handle, x: torch.Tensor, weights: Sequence[torch.Tensor], dy: torch.Tensor,
             want_dx: bool = True, want_dw=True, x_unchanged: bool = False, w_unchanged: bool = False):
    x = x.contiguous()
    dy = dy.contiguous()
    weights = [w.contiguous() for w in weights]
    code = _code([x, dy] + weights)
    if isinstance(want_dw, bool):
        want_dw = [want_dw] * len(weights)
    dx = torch.empty(h.x_shape, dtype=x.dtype, device=x.device) if want_dx else None
    dws = [torch.empty(tuple(s), dtype=x.dtype, device=x.device) if want_dw[j] else None
           for j, s in enumerate(h.w_shapes)]
    warr = (ctypes.c_void_p * max(1, len(weights)))(*[w.data_ptr() for w in weights])
    dwarr = (ctypes.c_void_p * max(1, len(weights)))(*[g.data_ptr() if g is not None else 0 for g in dws])
    with torch.cuda.device(x.device):
        rc = _lib.lib.syno_backward_ex(h.ptr, code, _ptr(x), warr, len(weights), _ptr(dy), _ptr(dx), dwarr,
                                       (_lib.SYNO_BWD_X_UNCHANGED if x_unchanged else 0)
                                       | (_lib.SYNO_BWD_W_UNCHANGED if w_unchanged else 0), _stream_ptr(x))
    if rc:
        raise_status(rc, _lib.last_error())
    return dx, dws


def index_map(h: Handle, term: int, coord: int, device=None) -> torch.Tensor:
    """K1 parity hook: raw coordinate values over the unstaged loop grid (int64)."""
    require_cuda()
    out = torch.empty(int(h.info.index_grid), dtype=torch.int64, device=device or torch.device("cuda"))
    rc = _lib.lib.syno_index_map(h.ptr, term, coord, _ptr(out),
                                 ctypes.c_void_p(torch.cuda.current_stream(out.device).cuda_stream))
    if rc:
        raise_status(rc, _lib.last_error())
    return out


class SynoFunction(torch.autograd.Function):
    """y = op(x, *weights) with the device backward (grad-input + grad-weight)."""

    @staticmethod
    def forward(ctx, h: Handle, x, *weights):
        ctx.h = h
        ctx.save_for_backward(x, *weights)
        return forward(h, x, list(weights))

    @staticmethod
    def backward(ctx, dy):
        x, *weights = ctx.saved_tensors
        need = ctx.needs_input_grad
        # autograd saved x and weights (version-checked), so the forward's
        # packed operands are reusable -- but only when the forward read these
        # very buffers: a non-contiguous operand was packed from a temporary
        # copy that is gone now, and the library's reuse check compares
        # pointers only (a new temporary may land at the freed address)
        dx, dws = backward(ctx.h, x, weights, dy, bool(need[1]), [bool(n) for n in need[2:]],
                           x_unchanged=x.is_contiguous(), w_unchanged=all(w.is_contiguous() for w in weights))
        return (None, dx, *dws)


class SynoOperator(torch.nn.Module):
    """A synthesized operator as a module: weights are parameters, N(0, std) init."""

    def __init__(self, graph, assignment: Optional[Mapping[str, int]] = None, staged: bool = False,
                 dtype=torch.bfloat16, device=None, std: Optional[float] = None, seed: int = 0):
        super().__init__()
        self.graph = graph
        self.h = handle_for(graph, assignment, staged)
        gen = torch.Generator(device="cpu").manual_seed(seed)
        self.weight = torch.nn.ParameterList()
        for shape in self.h.w_shapes:
            fan = max(1, int(np.prod(shape[1:])) if len(shape) > 1 else 1)
            s = std if std is not None else 1.0 / np.sqrt(fan)
            w = torch.randn(tuple(shape), generator=gen, dtype=torch.float32) * s
            self.weight.append(torch.nn.Parameter(w.to(device=device or "cuda", dtype=dtype)))

    def forward(self, x):
        return SynoFunction.apply(self.h, x, *self.weight)

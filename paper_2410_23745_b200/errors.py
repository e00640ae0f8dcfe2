"""Exceptions with the reference's names.

    ShapeMismatch       codegen.py:68
    NonIntegralSize     symexpr.py:21
    GraphError          pgraph.py:66
    OperatorParseError  pgraph.py:655 (a ValueError, as in the reference)
    LoopNestParseError  codegen.py:72 (a ValueError)
"""
from __future__ import annotations

from . import _lib


class ShapeMismatch(Exception):
    """An array does not have the shape the operator requires."""


class NonIntegralSize(Exception):
    """A size expression did not evaluate to a positive whole number."""


class GraphError(Exception):
    """Base for all graph construction failures."""


class OperatorParseError(ValueError):
    pass


class LoopNestParseError(ValueError):
    """Malformed loop-nest text (codegen.parse_loop_nest)."""


class UnsupportedOperator(Exception):
    """The operator exceeds a limit of the device engine (never a silent fallback)."""


class DeviceError(RuntimeError):
    """A CUDA runtime failure inside the native library."""


_BY_STATUS = {
    _lib.SYNO_E_PARSE: OperatorParseError,
    _lib.SYNO_E_GRAPH: GraphError,
    _lib.SYNO_E_SHAPE: ShapeMismatch,
    _lib.SYNO_E_NONINTEGRAL: NonIntegralSize,
    _lib.SYNO_E_KEY: KeyError,
    _lib.SYNO_E_VALUE: ValueError,
    _lib.SYNO_E_CUDA: DeviceError,
    _lib.SYNO_E_INVALID: ValueError,
    _lib.SYNO_E_UNSUPPORTED: UnsupportedOperator,
}


def raise_status(rc: int, message: str):
    raise _BY_STATUS.get(rc, RuntimeError)(message)

"""B200 execution backend for Syno synthesized operators (arXiv 2410.23745).

The reference ("opsmith") runs operators with a float64 numpy interpreter;
this package keeps its operator-construction and execution API
(pgraph / codegen) and runs them through sm_100a CUDA kernels in the
in-tree native library libsyno.so (C ABI: include/syno.h).
"""
from . import _lib  # noqa: F401  (fails loudly when libsyno.so is missing)
from .errors import (  # noqa: F401
    DeviceError, GraphError, NonIntegralSize, OperatorParseError, ShapeMismatch, UnsupportedOperator,
)
from .pgraph import (  # noqa: F401
    PGraph, ProblemSpec, Variable, build_spec, handle_for, operator_document, parse_operator, parse_steps,
    print_operator, print_steps,
)

__version__ = "0.1.0"

"""Operator-construction API mirror (reference: opsmith/pgraph.py).

The reference builds a ``PGraph`` in Python by replaying primitive steps
(pgraph.py:223-403).  Here the replay, lowering and planning happen in the
native library (csrc/graph.cpp, csrc/nest.cpp); this module keeps the
reference's names and argument meanings so caller code reads the same:

    spec = ProblemSpec(name, variables, reference, output_dims, input_dims, batch_dims)
    g = parse_steps("op{...}", spec)          # pgraph.py:675
    g = parse_operator(document)              # pgraph.py:730
    print_steps(g) / print_operator(g)        # pgraph.py:659 / 712

Sizes may be given as text ("C_in", "s*H", "K^2") or as any object whose
``str()`` is the reference's size text (e.g. the reference's own
``SymbolicSize``).  ``operator_document`` also accepts a reference
``PGraph`` object (duck-typed: ``.spec`` and ``.steps``), which is how the
reference's own graphs reach this backend.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from typing import Mapping, Optional

from . import _lib
from .errors import raise_status


@dataclass(frozen=True)
class Variable:
    name: str
    primary: bool = True


@dataclass(frozen=True)
class ProblemSpec:
    """pgraph.ProblemSpec (pgraph.py:127-158); search knobs are carried, not used."""

    name: str
    variables: tuple
    reference: tuple
    output_dims: tuple
    input_dims: tuple
    batch_dims: tuple = ()
    max_depth: int = 9
    flops_cap: Optional[int] = None
    params_cap: Optional[int] = None
    max_param_degree: int = 2
    max_expand: int = 2
    max_stride: int = 2

    @property
    def assignment(self) -> dict:
        return dict(self.reference)

    def header(self) -> str:
        ref = dict(self.reference)
        lines = [f"operator {self.name}"]
        for v in self.variables:
            kind = "primary" if v.primary else "coefficient"
            lines.append(f"var {v.name} {kind} {ref[v.name]}")
        lines.append("output " + " ".join(str(s) for s in self.output_dims))
        lines.append("input " + " ".join(str(s) for s in self.input_dims))
        if self.batch_dims:
            lines.append("batch " + " ".join(str(s) for s in self.batch_dims))
        return "\n".join(lines) + "\n"


def build_spec(name, primaries, coeffs, reference, output, input_, batch=(), **kw) -> ProblemSpec:
    """Convenience constructor with the reference tests' argument order
    (reference tests/conftest.py:14-27)."""
    variables = tuple(Variable(n) for n in primaries) + tuple(Variable(n, False) for n in coeffs)
    return ProblemSpec(name, variables, tuple(reference.items()), tuple(output), tuple(input_), tuple(batch), **kw)


@dataclass(frozen=True, eq=False)
class PGraph:
    """A replayed operator: its spec, its step string and its document."""

    spec: ProblemSpec
    steps_text: str
    document: str = field(repr=False)
    n_weights: int = 0
    complete: bool = True

    def __hash__(self):
        return hash(self.document)

    def __eq__(self, other):
        return isinstance(other, PGraph) and self.document == other.document


def _ref_step_text(step) -> str:
    """Text of one reference ``Step`` (pgraph.print_steps, pgraph.py:659-672)."""
    if step.kind == "reduce":
        return f"reduce({step.param})"
    if step.kind == "contract":
        return "contract[" + ",".join(f"{t}:{m}" for t, m in zip(step.targets, step.modes)) + "]"
    if step.kind in ("merge", "stride"):
        return f"{step.kind}({step.param})[{step.targets[0]}]"
    return f"{step.kind}[" + ",".join(str(t) for t in step.targets) + "]"


def print_steps(graph) -> str:
    if isinstance(graph, PGraph):
        return graph.steps_text
    return "op{" + "; ".join(_ref_step_text(s) for s in graph.steps) + "}"


def spec_header(spec) -> str:
    """The operator/var/output/input/batch lines of our ProblemSpec or of a
    reference ProblemSpec (pgraph.print_operator's header, pgraph.py:712-723)."""
    if isinstance(spec, ProblemSpec):
        return spec.header()
    ref = dict(spec.reference)
    lines = [f"operator {spec.name}"]
    for v in spec.variables:
        lines.append(f"var {v.name} {'primary' if v.primary else 'coefficient'} {ref[v.name]}")
    lines.append("output " + " ".join(str(s) for s in spec.output_dims))
    lines.append("input " + " ".join(str(s) for s in spec.input_dims))
    if spec.batch_dims:
        lines.append("batch " + " ".join(str(s) for s in spec.batch_dims))
    return "\n".join(lines) + "\n"


def operator_document(graph) -> str:
    """The operator document of our PGraph or of a reference PGraph."""
    if isinstance(graph, PGraph):
        return graph.document
    text = spec_header(graph.spec) + "steps " + print_steps(graph) + "\n"
    # the reference's print_operator ends with the match_input permutation
    # (pgraph.py:724-726); the native replay computes it (csrc/graph.cpp)
    with _CACHE_LOCK:
        doc = _REF_DOCS.get(text)
    if doc is None:
        doc = Handle(text, None, False, replay_only=True).document()
        with _CACHE_LOCK:
            if len(_REF_DOCS) >= _CACHE_MAX:
                _REF_DOCS.pop(next(iter(_REF_DOCS)))
            _REF_DOCS[text] = doc
    return doc


# ---------------------------------------------------------------------------
# Compiled handles, cached per (document, assignment, staged)
# ---------------------------------------------------------------------------

class Handle:
    """Owns one native syno_op_t."""

    def __init__(self, document: str, assignment: Optional[Mapping[str, int]], staged: bool,
                 replay_only: bool = False, nest_text: Optional[str] = None):
        kv = None
        if assignment is not None:
            kv = ",".join(f"{k}={int(v)}" for k, v in assignment.items()).encode()
        ptr = ctypes.c_void_p()
        if nest_text is not None:
            # codegen.parse_loop_nest: `document` only supplies the spec
            rc = _lib.lib.syno_compile_nest(document.encode(), nest_text.encode(), kv, 0, ctypes.byref(ptr))
        else:
            flags = (_lib.SYNO_STAGED if staged else 0) | (_lib.SYNO_REPLAY_ONLY if replay_only else 0)
            rc = _lib.lib.syno_compile(document.encode(), kv, flags, ctypes.byref(ptr))
        if rc:
            raise_status(rc, _lib.last_error())
        self.ptr = ptr
        info = _lib.SynoInfo()
        rc = _lib.lib.syno_query(self.ptr, ctypes.byref(info))
        if rc:
            raise_status(rc, _lib.last_error())
        self.info = info
        self.n_weights = info.n_weights
        self.x_shape = tuple(info.x_shape[k] for k in range(info.x_rank))
        self.y_shape = tuple(info.y_shape[k] for k in range(info.y_rank))
        self.w_shapes = [tuple(info.w_shape[j][k] for k in range(info.w_rank[j])) for j in range(info.n_weights)]
        self.batch_rank = info.batch_rank
        self.flops_unstaged = info.flops_unstaged
        self.flops_staged = info.flops_staged
        self.params = info.params

    def emit(self, staged: bool) -> str:
        return _lib.text_call(_lib.lib.syno_emit_loop_nest, self.ptr, int(staged))

    def describe(self) -> str:
        return _lib.text_call(_lib.lib.syno_describe_plan, self.ptr)

    def document(self) -> str:
        return _lib.text_call(_lib.lib.syno_print_operator, self.ptr)

    def __del__(self):
        ptr = getattr(self, "ptr", None)
        if ptr is not None and ptr.value and _lib is not None and _lib.lib is not None:
            _lib.lib.syno_destroy(ptr)
            self.ptr = None


_CACHE: dict = {}
_REF_DOCS: dict = {}
_CACHE_LOCK = threading.Lock()
_CACHE_MAX = 4096


def handle_for(graph, assignment: Optional[Mapping[str, int]] = None, staged: bool = False) -> Handle:
    doc = operator_document(graph)
    key = (doc, None if assignment is None else tuple(sorted((k, int(v)) for k, v in assignment.items())), bool(staged))
    with _CACHE_LOCK:
        h = _CACHE.get(key)
    if h is not None:
        return h
    h = Handle(doc, assignment, staged)
    with _CACHE_LOCK:
        if len(_CACHE) >= _CACHE_MAX:
            _CACHE.pop(next(iter(_CACHE)))
        _CACHE[key] = h
    return h


def _from_document(doc: str) -> PGraph:
    h = Handle(doc, None, False, replay_only=True)
    text = h.document()
    spec_lines = {}
    variables, reference = [], []
    steps = ""
    for line in text.splitlines():
        head, _, rest = line.partition(" ")
        if head == "var":
            name, kind, val = rest.split()
            variables.append(Variable(name, kind == "primary"))
            reference.append((name, int(val)))
        elif head in ("output", "input", "batch"):
            spec_lines[head] = tuple(rest.split())
        elif head == "operator":
            spec_lines["name"] = rest
        elif head == "steps":
            steps = rest
    spec = ProblemSpec(
        spec_lines["name"], tuple(variables), tuple(reference),
        spec_lines.get("output", ()), spec_lines.get("input", ()), spec_lines.get("batch", ()),
    )
    return PGraph(spec, steps, text, h.n_weights, bool(h.info.complete))


def parse_steps(text: str, spec: ProblemSpec) -> PGraph:
    """Replay a step string against a spec (pgraph.py:675-709).

    Raises OperatorParseError for malformed or unreplayable steps, as the
    reference does.  Graphs whose frontier does not match the input are
    returned too (complete=False); executing them raises ShapeMismatch.
    """
    g = _from_document(spec.header() + "steps " + text.strip() + "\n")
    return PGraph(spec, g.steps_text, g.document, g.n_weights, g.complete)


def parse_operator(doc: str) -> PGraph:
    """Parse a standalone operator document (pgraph.py:730-790)."""
    return _from_document(doc)


def print_operator(graph) -> str:
    if isinstance(graph, PGraph) and graph.complete:
        return graph.document
    return operator_document(graph)

"""The C-ABI library: loads, exports every symbol include/syno.h declares,
and its host-side logic (compile, query, text forms, plan derivation) works
without a GPU.  No compute entry point is called here."""
from __future__ import annotations

import ctypes
import os
import re

from conftest import ROOT

from paper_2410_23745_b200 import _lib
from paper_2410_23745_b200 import pgraph as P

CONV = ("op{reduce(C_in); reduce(K); reduce(K); contract[0:weight,3:both,4:both,5:both]; "
        "unfold[1,7]; unfold[2,8]}")


def declared_functions():
    text = open(os.path.join(ROOT, "include", "syno.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(syno_\w+)\s*\(", text, re.M)))


def test_header_and_library_agree():
    names = declared_functions()
    assert set(names) == set(_lib.EXPORTS), names
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n


def test_library_is_in_tree_and_versioned():
    assert os.path.dirname(_lib.LIB_PATH) == os.path.join(ROOT, "paper_2410_23745_b200")
    assert b"sm_100a" in _lib.lib.syno_version()


def conv_spec(batch=True):
    return P.build_spec("conv", ("C_out", "C_in", "H", "W") + (("N",) if batch else ()), ("K",),
                        {"C_out": 64, "C_in": 64, "H": 32, "W": 32, "K": 3, **({"N": 8} if batch else {})},
                        ("C_out", "H", "W"), ("C_in", "H", "W"), ("N",) if batch else ())


def test_query_shapes_and_flops():
    g = P.parse_steps(CONV, conv_spec())
    h = P.handle_for(g)
    assert h.x_shape == (8, 64, 32, 32) and h.y_shape == (8, 64, 32, 32)
    assert h.w_shapes == [(64, 64, 3, 3)]
    assert h.flops_unstaged == 603979776 == h.flops_staged
    assert h.params == 64 * 64 * 9


def test_gradient_plans_are_gather_form_for_the_conv_family():
    """grad-input of a conv inverts to a transposed gather (no atomics);
    grad-weight indexes the weight by bare iterators."""
    for steps in (CONV,
                  "op{reduce(C_in); contract[0:weight,3:both]}",
                  "op{reduce(C_in); reduce(K); reduce(K); contract[0:weight,3:both,4:both]; unfold[1,7]; "
                  "contract[5:both]; unfold[2,9]}"):
        h = P.handle_for(P.parse_steps(steps, conv_spec()))
        assert h.info.grad_x_scatter == 0, steps
        assert all(h.info.grad_w_scatter[j] == 0 for j in range(h.n_weights)), steps
        text = h.describe()
        assert text.count("gather") >= 2


def test_replay_only_handles_refuse_execution():
    h = P.Handle(P.parse_steps(CONV, conv_spec()).document, None, False, replay_only=True)
    assert h.info.complete == 1 and h.info.replay_only == 1
    rc = _lib.lib.syno_forward(h.ptr, 0, ctypes.c_void_p(1), None, 0, ctypes.c_void_p(1), None)
    assert rc == _lib.SYNO_E_SHAPE or rc == _lib.SYNO_E_INVALID


def test_bad_arguments_report_status_and_message():
    ptr = ctypes.c_void_p()
    rc = _lib.lib.syno_compile(b"operator x\nsteps op{}\n", None, 0, ctypes.byref(ptr))
    assert rc == _lib.SYNO_E_PARSE
    assert "output and input" in _lib.last_error()
    rc = _lib.lib.syno_compile(None, None, 0, ctypes.byref(ptr))
    assert rc == _lib.SYNO_E_INVALID


def test_config_operators_take_the_tensor_core_path():
    """Host-side matcher: every Appendix-A contraction operator qualifies
    for the tcgen05 path; pooling (no weights) stays on the universal engine."""
    from paper_2410_23745_b200 import workloads as WL
    for L in WL.resnet18_cifar(8) + [WL.qkv(2, 64), WL.cfg1_conv(2)]:
        assert P.handle_for(L.graph).info.tc_path == 1, L.name
    pool = P.parse_steps(WL.SUMPOOL3X3, P.build_spec("pool", ("C", "H", "W", "N"), ("K",),
                                                     {"C": 8, "H": 8, "W": 8, "N": 2, "K": 3},
                                                     ("C", "H", "W"), ("C", "H", "W"), ("N",)))
    assert P.handle_for(pool).info.tc_path == 0

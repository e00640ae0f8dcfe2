"""The BASELINE.json config set as plain data.

Pure Python with no package-relative imports and no native library, so the
reference arm of bench.py can load this file by path and build the SAME
operators with the reference's own ``opsmith.pgraph.parse_steps`` without
ever loading libsyno.so.  ``workloads.py`` builds the backend's graphs from
the same tables.

Operator step strings are the verified set of SURVEY Appendix A (each
replays and passes the reference's canonicality check).
"""
from __future__ import annotations

import os

CONV3X3 = ("op{reduce(C_in); reduce(K); reduce(K); contract[0:weight,3:both,4:both,5:both]; "
           "unfold[1,7]; unfold[2,8]}")
CONV3X3_S2 = ("op{reduce(C_in); reduce(K); reduce(K); contract[0:weight,3:both,4:both,5:both]; "
              "stride(s)[1]; unfold[9,7]; stride(s)[2]; unfold[11,8]}")
SEP_SHARED = ("op{reduce(C_in); reduce(K); reduce(K); contract[0:weight,3:both,4:both]; "
              "unfold[1,7]; contract[5:both]; unfold[2,9]}")
POINTWISE = "op{reduce(C_in); contract[0:weight,3:both]}"
SUMPOOL3X3 = "op{reduce(K); reduce(K); unfold[1,3]; unfold[2,4]}"
QKV = "op{reduce(E); contract[1:weight,2:both]}"

STEPS = {"conv3x3": CONV3X3, "conv3x3_s2": CONV3X3_S2, "sep_shared": SEP_SHARED, "pointwise": POINTWISE,
         "shortcut_s2": CONV3X3_S2, "qkv": QKV}


def conv_spec_args(name: str, op: str, c_in: int, c_out: int, h: int, batch: int):
    """(name, primaries, coefficients, reference, output, input, batch) of a
    conv-spec layer: output (C_out, H, W), input (C_in, [s*]H, [s*]W), batch (N)."""
    strided = op in ("conv3x3_s2", "shortcut_s2")
    k = 1 if op == "shortcut_s2" else 3
    ref = {"C_out": c_out, "C_in": c_in, "H": h, "W": h, "N": batch, "K": k}
    coeffs = ("K",)
    if strided:
        ref["s"] = 2
        coeffs = ("K", "s")
    return (name, ("C_out", "C_in", "H", "W", "N"), coeffs, ref, ("C_out", "H", "W"),
            ("C_in", "s*H", "s*W") if strided else ("C_in", "H", "W"), ("N",))


def qkv_spec_args(batch: int = 16, t: int = 1024, e: int = 768, e3: int = 2304):
    ref = {"T": t, "E": e, "E3": e3, "B": batch}
    return ("qkv", ("T", "E", "E3", "B"), (), ref, ("T", "E3"), ("T", "E"), ("B",))


def resnet18_table():
    """cfg2: (name, op, c_in, c_out, h) of the 20 conv layers of ResNet-18
    (CIFAR variant, 32x32).  Stride-1 3x3 convs alternate sep_shared (the
    paper's Operator-2-like shared-weight op) and conv3x3; stride-2 convs are
    conv3x3_s2; the 1x1 stride-2 shortcuts are the strided op with K=1."""
    rows = [("stem", "conv3x3", 3, 64, 32)]
    cin = 64
    for stage, (c, h) in enumerate(((64, 32), (128, 16), (256, 8), (512, 4)), start=1):
        for blk in range(2):
            first = blk == 0 and stage > 1
            rows.append((f"l{stage}b{blk}c1", "conv3x3_s2" if first else "sep_shared", cin, c, h))
            rows.append((f"l{stage}b{blk}c2", "conv3x3", c, c, h))
            if first:
                rows.append((f"l{stage}b{blk}sc", "shortcut_s2", cin, c, h))
            cin = c
    return rows


def resnet34_table():
    """cfg3: ResNet-34 stages at 224x224 input (56/28/14/7 feature maps)."""
    rows = []
    cin = 64
    for stage, (c, h, n) in enumerate(((64, 56, 3), (128, 28, 4), (256, 14, 6), (512, 7, 3)), start=1):
        for blk in range(n):
            first = blk == 0 and stage > 1
            rows.append((f"l{stage}b{blk}c1", "conv3x3_s2" if first else "sep_shared", cin, c, h))
            rows.append((f"l{stage}b{blk}c2", "conv3x3", c, c, h))
            if first:
                rows.append((f"l{stage}b{blk}sc", "shortcut_s2", cin, c, h))
            cin = c
    return rows


CORPUS_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                           "corpus_conv64.txt")
CORPUS_REF = {"C_out": 64, "C_in": 64, "H": 32, "W": 32, "K": 3, "s": 2}


QKV_CORPUS_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                               "corpus_qkv.txt")


def qkv_variant_ops():
    """cfg4's sampled variants of the QKV projection: the dense
    baseline first, then operators the reference sampler drew on the QKV spec
    within 2x its FLOPs and parameters (tests/golden/make_qkv_corpus.py)."""
    return [ln.strip() for ln in open(QKV_CORPUS_PATH) if ln.strip()]


def corpus_ops(limit=None):
    ops = [ln.strip() for ln in open(CORPUS_PATH) if ln.strip()]
    return ops[:limit] if limit is not None else ops


def corpus_spec_args(batch: int = 8):
    ref = dict(CORPUS_REF, N=batch)
    return ("conv64", ("C_out", "C_in", "H", "W", "N"), ("K", "s"), ref, ("C_out", "H", "W"), ("C_in", "H", "W"),
            ("N",))

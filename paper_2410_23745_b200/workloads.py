"""The BASELINE.json config set as operator documents.

cfg1  conv3x3 N=8 C=64 H=W=32, fp32, forward
cfg2  ResNet-18 CIFAR-shape conv layers, each replaced by a synthesized
      operator, fwd+bwd bf16 batch 128
cfg3  ResNet-34 ImageNet-shape layers, fwd+bwd bf16 batch 256
cfg4  GPT-2-small QKV projection as a synthesized operator, B=16 T=1024
cfg5  the 1024-operator sampled corpus (tests/golden/corpus_conv64.txt)

Operator step strings are the verified set of SURVEY Appendix A (each
replays and passes the reference's canonicality check).
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

from .pgraph import PGraph, build_spec, parse_steps

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
         "shortcut_s2": CONV3X3_S2}


@dataclass(frozen=True)
class Layer:
    name: str
    op: str            # key of STEPS
    graph: PGraph
    assignment: dict

    @property
    def steps(self) -> str:
        return STEPS[self.op]


def conv_layer(name: str, op: str, c_in: int, c_out: int, h: int, batch: int) -> Layer:
    """A conv-spec layer: output (C_out, H, W), input (C_in, [s*]H, [s*]W), batch (N)."""
    strided = op in ("conv3x3_s2", "shortcut_s2")
    k = 1 if op == "shortcut_s2" else 3
    ref = {"C_out": c_out, "C_in": c_in, "H": h, "W": h, "N": batch, "K": k}
    coeffs = ("K",)
    if strided:
        ref["s"] = 2
        coeffs = ("K", "s")
    spec = build_spec(f"{name}", ("C_out", "C_in", "H", "W", "N"), coeffs, ref,
                      ("C_out", "H", "W"), ("C_in", "s*H", "s*W") if strided else ("C_in", "H", "W"), ("N",))
    return Layer(name, op, parse_steps(STEPS[op], spec), ref)


def resnet18_cifar(batch: int = 128) -> list:
    """cfg2: the 20 conv layers of ResNet-18 (CIFAR variant, 32x32), every one a
    synthesized operator.  Stride-1 3x3 convs alternate sep_shared (the
    paper's Operator-2-like shared-weight op) and conv3x3; stride-2 convs are
    conv3x3_s2; the 1x1 stride-2 shortcuts are the strided op with K=1."""
    layers = [conv_layer("stem", "conv3x3", 3, 64, 32, batch)]
    cin = 64
    for stage, (c, h) in enumerate(((64, 32), (128, 16), (256, 8), (512, 4)), start=1):
        for blk in range(2):
            first = blk == 0 and stage > 1
            layers.append(conv_layer(f"l{stage}b{blk}c1", "conv3x3_s2" if first else "sep_shared",
                                     cin, c, h, batch))
            layers.append(conv_layer(f"l{stage}b{blk}c2", "conv3x3", c, c, h, batch))
            if first:
                layers.append(conv_layer(f"l{stage}b{blk}sc", "shortcut_s2", cin, c, h, batch))
            cin = c
    return layers


def resnet34_imagenet(batch: int = 256) -> list:
    """cfg3: ResNet-34 stages at 224x224 input (56/28/14/7 feature maps)."""
    layers = []
    cin = 64
    for stage, (c, h, n) in enumerate(((64, 56, 3), (128, 28, 4), (256, 14, 6), (512, 7, 3)), start=1):
        for blk in range(n):
            first = blk == 0 and stage > 1
            layers.append(conv_layer(f"l{stage}b{blk}c1", "conv3x3_s2" if first else "sep_shared",
                                     cin, c, h, batch))
            layers.append(conv_layer(f"l{stage}b{blk}c2", "conv3x3", c, c, h, batch))
            if first:
                layers.append(conv_layer(f"l{stage}b{blk}sc", "shortcut_s2", cin, c, h, batch))
            cin = c
    return layers


def cfg1_conv(batch: int = 8) -> Layer:
    return conv_layer("cfg1_conv3x3", "conv3x3", 64, 64, 32, batch)


def qkv(batch: int = 16, t: int = 1024, e: int = 768, e3: int = 2304) -> Layer:
    ref = {"T": t, "E": e, "E3": e3, "B": batch}
    spec = build_spec("qkv", ("T", "E", "E3", "B"), (), ref, ("T", "E3"), ("T", "E"), ("B",))
    return Layer("qkv", "qkv", parse_steps(QKV, spec), ref)


STEPS["qkv"] = QKV

CORPUS_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                           "corpus_conv64.txt")


def corpus(batch: int = 8, limit: Optional[int] = None) -> list:
    """cfg5: the sampled corpus replayed with a batch dim on the conv64 spec."""
    ops = [ln.strip() for ln in open(CORPUS_PATH) if ln.strip()]
    if limit is not None:
        ops = ops[:limit]
    ref = {"C_out": 64, "C_in": 64, "H": 32, "W": 32, "K": 3, "s": 2, "N": batch}
    spec = build_spec("conv64", ("C_out", "C_in", "H", "W", "N"), ("K", "s"), ref,
                      ("C_out", "H", "W"), ("C_in", "H", "W"), ("N",))
    return [parse_steps(op, spec) for op in ops]

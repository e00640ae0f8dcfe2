"""The BASELINE.json config set as backend graphs.

cfg1  conv3x3 N=8 C=64 H=W=32, fp32, forward
cfg2  ResNet-18 CIFAR-shape conv layers, each replaced by a synthesized
      operator, fwd+bwd bf16 batch 128
cfg3  ResNet-34 ImageNet-shape layers, fwd+bwd bf16 batch 256
cfg4  GPT-2-small QKV projection as a synthesized operator, B=16 T=1024
cfg5  the 1024-operator sampled corpus (tests/golden/corpus_conv64.txt)

The tables and step strings live in ``configs.py`` (plain data, shared
with the reference arm of bench.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

from .configs import (  # noqa: F401  (re-exported names)
    CONV3X3, CONV3X3_S2, CORPUS_PATH, POINTWISE, QKV, SEP_SHARED, STEPS, SUMPOOL3X3, conv_spec_args,
    corpus_ops, corpus_spec_args, qkv_spec_args, qkv_variant_ops, resnet18_table, resnet34_table,
)
from .pgraph import PGraph, build_spec, parse_steps


@dataclass(frozen=True)
class Layer:
    name: str
    op: str            # key of STEPS
    graph: PGraph
    assignment: dict

    @property
    def steps(self) -> str:
        return STEPS.get(self.op, self.op)


def conv_layer(name: str, op: str, c_in: int, c_out: int, h: int, batch: int) -> Layer:
    """A conv-spec layer: output (C_out, H, W), input (C_in, [s*]H, [s*]W), batch (N)."""
    args = conv_spec_args(name, op, c_in, c_out, h, batch)
    return Layer(name, op, parse_steps(STEPS[op], build_spec(*args)), args[3])


def resnet18_cifar(batch: int = 128) -> list:
    return [conv_layer(n, op, ci, co, h, batch) for n, op, ci, co, h in resnet18_table()]


def resnet34_imagenet(batch: int = 256) -> list:
    return [conv_layer(n, op, ci, co, h, batch) for n, op, ci, co, h in resnet34_table()]


def cfg1_conv(batch: int = 8) -> Layer:
    return conv_layer("cfg1_conv3x3", "conv3x3", 64, 64, 32, batch)


def qkv(batch: int = 16, t: int = 1024, e: int = 768, e3: int = 2304) -> Layer:
    args = qkv_spec_args(batch, t, e, e3)
    return Layer("qkv", "qkv", parse_steps(QKV, build_spec(*args)), args[3])


def qkv_variants(batch: int = 16, t: int = 1024) -> list:
    """cfg4: the dense QKV projection and its sampled variants (one Layer each,
    op = the step string)."""
    args = qkv_spec_args(batch, t)
    spec = build_spec(*args)
    return [Layer(f"qkv_v{i}", op, parse_steps(op, spec), args[3]) for i, op in enumerate(qkv_variant_ops())]


def corpus(batch: int = 8, limit: Optional[int] = None) -> list:
    """cfg5: the sampled corpus replayed with a batch dim on the conv64 spec."""
    spec = build_spec(*corpus_spec_args(batch))
    return [parse_steps(op, spec) for op in corpus_ops(limit)]

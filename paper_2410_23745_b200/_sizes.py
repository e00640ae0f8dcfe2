"""Size text evaluation for shape helpers (symexpr.eval_size, symexpr.py:103-121)."""
from __future__ import annotations

from typing import Mapping

from .errors import NonIntegralSize


def eval_size_text(text: str, env: Mapping[str, int]) -> int:
    text = text.strip()
    if text == "1":
        return 1
    num, den = 1, 1
    for factor in text.split("*"):
        name, _, exp_text = factor.strip().partition("^")
        exp = int(exp_text) if exp_text else 1
        val = env[name.strip()]
        if val < 1:
            raise ValueError(f"assignment for {name} must be >= 1, got {val}")
        if exp > 0:
            num *= val ** exp
        else:
            den *= val ** (-exp)
    if num % den:
        raise NonIntegralSize(f"{text} is not integral under {dict(env)}")
    return num // den

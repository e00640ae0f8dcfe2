"""The reference's tensor file format (codegen.py:950-976) in the native
library, and the spec'd `emit` CLI.  CPU only: neither
touches the device.  Mirrors reference tests/test_codegen.py:451-474 and pins
byte equality against files written by the reference itself."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import CASES, GOLDEN, ROOT

from paper_2410_23745_b200.codegen import load_tensor, save_tensor
from paper_2410_23745_b200.errors import ShapeMismatch


def test_tensor_round_trip_and_layout(tmp_path):
    rng = np.random.default_rng(21)
    arr = rng.standard_normal((2, 3, 4))
    path = tmp_path / "t.tensor"
    save_tensor(path, arr)
    raw = path.read_bytes()
    header = np.frombuffer(raw[: 8 * 4], dtype="<i8")
    assert list(header) == [3, 2, 3, 4]
    assert len(raw) == 8 * 4 + 8 * 24
    first = np.frombuffer(raw[32:64], dtype="<f8")
    assert np.array_equal(first, arr[0, 0])
    assert np.array_equal(load_tensor(path), arr)


def test_tensor_scalar_and_truncation(tmp_path):
    path = tmp_path / "s.tensor"
    save_tensor(path, np.float64(4.25))
    back = load_tensor(path)
    assert back.shape == ()
    assert back == 4.25
    path.write_bytes(path.read_bytes()[:-4])
    with pytest.raises(ShapeMismatch):
        load_tensor(path)
    (tmp_path / "h.tensor").write_bytes(b"\x01\x00")
    with pytest.raises(ShapeMismatch):
        load_tensor(tmp_path / "h.tensor")


@pytest.mark.parametrize("name,shape", [("ref_3d", (2, 3, 4)), ("ref_scalar", ())])
def test_reference_written_files(tmp_path, name, shape):
    ref = os.path.join(GOLDEN, f"{name}.tensor")
    arr = load_tensor(ref)
    assert arr.shape == shape
    out = tmp_path / "copy.tensor"
    save_tensor(out, arr)
    assert out.read_bytes() == open(ref, "rb").read()


def test_cli_emit_matches_reference_nest(tmp_path):
    case = next(c for c in CASES if c["name"] == "conv2d_8")
    op = tmp_path / "op.txt"
    op.write_text(case["document"])
    out = tmp_path / "nest.txt"
    r = subprocess.run([sys.executable, "-m", "paper_2410_23745_b200", "emit", "--op", str(op), "--output", str(out)],
                       cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert out.read_text() == case["nest"]


def test_cli_config_error_exit_code(tmp_path):
    bad = tmp_path / "bad.txt"
    bad.write_text("operator x\nsteps op{bogus}\n")
    r = subprocess.run([sys.executable, "-m", "paper_2410_23745_b200", "emit", "--op", str(bad)],
                       cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert r.returncode == 2

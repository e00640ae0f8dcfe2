"""Golden .tensor files written by the REFERENCE's codegen.save_tensor.

Test infrastructure only (this container only: imports /root/reference).
Writes tests/golden/ref_{3d,scalar}.tensor; tests/test_tensor_io.py checks
that the backend reads them and writes byte-identical files.

    python tests/golden/make_tensor_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from opsmith.codegen import save_tensor  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(21)
save_tensor(os.path.join(HERE, "ref_3d.tensor"), rng.standard_normal((2, 3, 4)))
save_tensor(os.path.join(HERE, "ref_scalar.tensor"), np.float64(4.25))
print("ok")

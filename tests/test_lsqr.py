"""CPU: the LSQR restatement used by the device reward (reward.lsqr_device)
against scipy.sparse.linalg.lsqr, the solver the reference calls
(reward.py:128).  lsqr_device only needs matvec / rmatvec and torch vector
ops, so it runs on CPU tensors here and on device tensors in the reward."""
from __future__ import annotations

import numpy as np
import pytest
import torch
from scipy.sparse.linalg import lsqr

from paper_2410_23745_b200.reward import lsqr_device


@pytest.mark.parametrize("m,n,seed", [(40, 10, 0), (30, 30, 1), (12, 25, 2), (200, 50, 3)])
def test_lsqr_matches_scipy(m, n, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n))
    b = rng.standard_normal(m)
    want = lsqr(A, b, atol=1e-10, btol=1e-10, iter_lim=max(2 * n, 40))[0]
    At = torch.from_numpy(A)
    got, istop, itn = lsqr_device(lambda v: At @ v, lambda u: At.T @ u, torch.from_numpy(b), n,
                                  atol=1e-10, btol=1e-10, iter_lim=max(2 * n, 40))
    assert istop != 0 and itn >= 1
    np.testing.assert_allclose(got.numpy(), want, rtol=1e-7, atol=1e-9)


def test_lsqr_consistent_system_exact():
    rng = np.random.default_rng(5)
    A = rng.standard_normal((20, 8))
    x = rng.standard_normal(8)
    At = torch.from_numpy(A)
    got, _, _ = lsqr_device(lambda v: At @ v, lambda u: At.T @ u, At @ torch.from_numpy(x), 8)
    np.testing.assert_allclose(got.numpy(), x, rtol=1e-8, atol=1e-10)


def test_lsqr_zero_rhs():
    At = torch.eye(3, dtype=torch.float64)
    got, istop, itn = lsqr_device(lambda v: At @ v, lambda u: At.T @ u, torch.zeros(3, dtype=torch.float64), 3)
    assert itn == 0 and float(got.abs().max()) == 0.0

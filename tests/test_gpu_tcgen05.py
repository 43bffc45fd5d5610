"""GPU: the tcgen05 operand-layout conventions (csrc/tc.cuh) on the device.

Y0 = A B^T (K-major A and B), Y1 = A B (MN-major B), Y2 = A^T X (MN-major A and B, K = 128
samples accumulated in TMEM), each a 3-term split-bf16 product with fp32 accumulation; checked
against fp64 numpy with an error bound relative to sum |a_k b_k| (split-bf16: <= ~2^-15)."""
import ctypes as C

import numpy as np
import pytest

from paper_2405_04416_b200 import dg

pytestmark = pytest.mark.gpu


def test_tcgen05_layouts_and_split_bf16():
    rng = np.random.default_rng(0)
    A = rng.normal(size=(128, 64)).astype(np.float32)
    B = rng.normal(size=(64, 64)).astype(np.float32)
    X = rng.normal(size=(128, 32)).astype(np.float32)
    Y0 = np.zeros((128, 64), np.float32)
    Y1 = np.zeros((128, 64), np.float32)
    Y2 = np.zeros((64, 32), np.float32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    rc = dg.lib().dg_selftest_tcgen05(p(A), p(B), p(X), p(Y0), p(Y1), p(Y2))
    assert rc == 0, dg.lib().dg_last_error()
    A64, B64, X64 = A.astype(np.float64), B.astype(np.float64), X.astype(np.float64)
    for got, ref, scale in ((Y0, A64 @ B64.T, np.abs(A64) @ np.abs(B64.T)),
                            (Y1, A64 @ B64, np.abs(A64) @ np.abs(B64)),
                            (Y2, A64.T @ X64, np.abs(A64.T) @ np.abs(X64))):
        err = np.abs(got - ref) / scale
        assert err.max() < 3e-5, err.max()

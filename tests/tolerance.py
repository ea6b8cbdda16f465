"""Tolerances used by the parity tests (readings Q11/Q12).

north_star: fp32 reductions pass at max relative error 1e-5 with an absolute floor of
1e-6, i.e. |got - ref| <= 1e-5 |ref| + 1e-6 elementwise.  For signed data (grad_out,
U(-1,1) features) the relative form is ill-posed where the sum cancels, so those tests
use the conditioned summation bound |got - ref| <= 1e-5 * S + 1e-6 with
S = sum |terms| computed by the oracle (reading Q11).  max/argmax, degrees, indices and
collate outputs are compared exactly.
"""
import numpy as np

RTOL = 1e-5
ATOL = 1e-6


def check_close(got, ref, abs_sum=None, rtol=RTOL, atol=ATOL, what="values"):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    scale = np.abs(ref) if abs_sum is None else np.asarray(abs_sum, np.float64)
    err = np.abs(got - ref)
    bound = rtol * scale + atol
    bad = err > bound
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError(
            f"{what}: {int(bad.sum())}/{bad.size} outside tolerance; first {idx.tolist()}: "
            f"got {got[tuple(idx[0])]!r} ref {ref[tuple(idx[0])]!r} bound {bound[tuple(idx[0])]!r}")
    return float((err / np.maximum(scale, 1e-30)).max()) if err.size else 0.0


def check_exact(got, ref, what="values"):
    got = np.asarray(got)
    ref = np.asarray(ref)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    if not np.array_equal(got, ref):
        bad = np.argwhere(got != ref)[:5]
        raise AssertionError(f"{what}: {int((got != ref).sum())} mismatches; first {bad.tolist()}: "
                             f"got {got[tuple(bad[0])]!r} ref {ref[tuple(bad[0])]!r}")

"""GPU: device math used by the kernels, against numpy / the CUDA library."""
import ctypes as C

import numpy as np
import pytest

from paper_2310_16668_b200 import _abi

pytestmark = pytest.mark.gpu


def test_fast_sincos_within_two_ulp():
    # kappa * r in every configuration is well inside [0, 1e3]; cover negative
    # and larger arguments of the supported range (|x| <= 2^20) too
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.uniform(0, 20, 200000), rng.uniform(-1e3, 1e3, 200000),
                        rng.uniform(-1e6, 1e6, 50000),
                        np.arange(-64, 65) * (np.pi / 4)]).astype(np.float64)
    out = np.zeros(6 * x.size)
    assert _abi.probe_lib().sfmm_probe_test_sincos(x.ctypes.data, x.size, out.ctypes.data) == 0
    s_ref, c_ref = out[4::6], out[5::6]
    assert np.allclose(s_ref, np.sin(x), atol=1e-15, rtol=0)
    # branch-free (out[0:2]) and table-driven (out[2:4]) versions: absolute
    # error <= 2 ulp of 1 (results are bounded by 1 in magnitude); the table
    # version is used only for |x| <= 2e4 (kSinCosTabMaxArg)
    tab_ok = np.abs(x) <= 2e4
    for s, c, m in ((out[0::6], out[1::6], np.ones_like(tab_ok)), (out[2::6], out[3::6], tab_ok)):
        assert np.max(np.abs(s - s_ref)[m]) <= 2 * np.spacing(1.0)
        assert np.max(np.abs(c - c_ref)[m]) <= 2 * np.spacing(1.0)
        assert np.max(np.abs(s - np.sin(x))[m]) <= 4 * np.spacing(1.0)
        assert np.max(np.abs(c - np.cos(x))[m]) <= 4 * np.spacing(1.0)


def test_table_log_within_two_ulp():
    # log(r^2) of the Laplace-2D kernels: squared distances span many decades,
    # with extra samples around 1 (no cancellation allowed there) and the
    # special inputs that must keep the library's behaviour
    rng = np.random.default_rng(6)
    x = np.concatenate([10.0 ** rng.uniform(-300, 300, 200000), rng.uniform(0.5, 2.0, 200000),
                        1.0 + rng.uniform(-1e-6, 1e-6, 50000), 1.0 + np.arange(-50, 51) * 2.0 ** -52,
                        np.array([1.0, 2.0, 0.5, np.sqrt(2.0), 1e-310, 0.0, np.inf])])
    out = np.zeros(2 * x.size)
    assert _abi.probe_lib().sfmm_probe_test_log(x.ctypes.data, x.size, out.ctypes.data) == 0
    got, ref = out[0::2], out[1::2]
    with np.errstate(divide="ignore"):
        assert np.allclose(ref, np.log(x), rtol=1e-15, atol=0, equal_nan=True)
    fin = np.isfinite(ref) & (ref != 0)
    rel = np.abs(got[fin] - ref[fin]) / np.abs(ref[fin])
    assert rel.max() <= 2 * np.spacing(1.0), rel.max()
    assert got[x == 1.0].tolist() == [0.0] * int((x == 1.0).sum())
    assert np.isneginf(got[x == 0.0]).all() and np.isposinf(got[x == np.inf]).all()

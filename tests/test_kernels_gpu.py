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
    out = np.zeros(4 * x.size)
    assert _abi.gpu_lib().sfmm_gpu_test_sincos(x.ctypes.data, x.size, out.ctypes.data) == 0
    s, c, s_ref, c_ref = out[0::4], out[1::4], out[2::4], out[3::4]
    assert np.allclose(s_ref, np.sin(x), atol=1e-15, rtol=0)
    # absolute error <= 2 ulp of 1 (results are bounded by 1 in magnitude)
    assert np.max(np.abs(s - s_ref)) <= 2 * np.spacing(1.0)
    assert np.max(np.abs(c - c_ref)) <= 2 * np.spacing(1.0)
    assert np.max(np.abs(s - np.sin(x))) <= 4 * np.spacing(1.0)
    assert np.max(np.abs(c - np.cos(x))) <= 4 * np.spacing(1.0)

"""The accurate log table of the 2D kernels (csrc/log_table.inc, tools/gen_log_table.py).

log_tab (csrc/fastmath.cuh) drops the low-order table term, which is exact only if
every v_k = -log(inv_k) - (k >= 53 ? ln2 : 0) is within a tiny fraction of an ulp of
its double; it also relies on inv_k staying close to 1/c_k so |t| stays below 1/128
(+ slack) for the degree-8 log1p.  Both properties are checked here at 160 bits.
"""
from __future__ import annotations

import math
import os
import re

import pytest

mpmath = pytest.importorskip("mpmath")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2310_16668_b200", "csrc")
# (file, entries, first right-end entry): fastmath.cuh SFMM_LOG_BITS = 7 / 9
TABLES = [("log_table.inc", 128, 53), ("log_table512.inc", 512, 213)]


def _entries(inc):
    pat = re.compile(r"\{\s*([-0-9a-fx.p+]+),\s*([-0-9a-fx.p+]+)\s*\}")
    out = []
    with open(os.path.join(CSRC, inc)) as f:
        for line in f:
            m = pat.search(line)
            if m:
                out.append((float.fromhex(m.group(1)), float.fromhex(m.group(2))))
    return out


@pytest.mark.parametrize("inc,size,split", TABLES)
def test_log_table_is_accurate(inc, size, split):
    mpmath.mp.prec = 160
    ln2 = mpmath.log(2)
    tab = _entries(inc)
    assert len(tab) == size
    for k, (inv, v) in enumerate(tab):
        upper = k >= split
        c = mpmath.mpf(1) + mpmath.mpf(k + 1 if upper else k) / size
        # inv within 2^-24 (relative) of 1/c: |t| < 1/size + 2^-23 on the entry's interval
        assert abs(mpmath.mpf(inv) * c - 1) < mpmath.mpf(2) ** -24, k
        exact = -mpmath.log(mpmath.mpf(inv)) - (ln2 if upper else 0)
        if v == 0.0:
            assert exact == 0, k
            continue
        err_ulp = abs(exact - mpmath.mpf(v)) / math.ulp(v)
        assert err_ulp < mpmath.mpf(2) ** -12, (k, float(err_ulp))
        # right ends carry v <= 0 and left ends v >= 0, so v and log1p(t) never cancel
        assert (v <= 0.0) if upper else (v >= 0.0), k

"""GPU tree and neighbor lists: bit-identical to the
host builder (itself pinned against the reference in tests/test_host.py) and
to the reference directly, as test_tree.cpp:168-200 pins the reference's own
tree; error behaviour as tree.cpp:148-186."""
import numpy as np
import pytest

from conftest import requires_ref
from oracle import pyoracle as po
from paper_2310_16668_b200 import api, host

pytestmark = pytest.mark.gpu

TREE_KEYS = ["pts", "perm", "level_begin", "box_parent", "box_level", "box_begin", "box_end",
             "box_leaf", "coll_off", "coll", "coarse_off", "coarse", "fine_off", "fine"]


def _geometry(hp):
    nb = hp.desc_struct().n_boxes
    c, h = np.zeros(3 * nb), np.zeros(nb)
    host._check(host.host_lib().sfmm_host_box_geometry(hp._h, c.ctypes.data, h.ctypes.data))
    return c, h


def _same_tree(pts, leaf):
    g = host.HostPlan.build_tree_gpu(pts, leaf)
    h = host.HostPlan.build_tree(pts, leaf)
    dg, dh = g.descriptor(), h.descriptor()
    for k in TREE_KEYS:
        assert np.array_equal(dg.arrays[k], dh.arrays[k]), k
    assert dg.scalars["depth"] == dh.scalars["depth"]
    cg, hg = _geometry(g)
    ch, hh = _geometry(h)
    assert np.array_equal(cg, ch) and np.array_equal(hg, hh)
    return dg


def _gaussian(n, seed=1, sigma=0.02):
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.1, 0.9, size=(16, 3))
    return centres[rng.integers(0, 16, n)] + sigma * rng.standard_normal((n, 3))


@pytest.mark.parametrize("dist,n,leaf", [
    ("square", 4000, 20), ("annulus", 8000, 50), ("cube", 5000, 60), ("sphere", 5000, 60),
    ("sphere", 30000, 30), ("cube", 60000, 128), ("annulus", 3000, 1), ("cube", 7, 1),
    ("cube", 1, 1), ("square", 100, 1000), ("cube", 5000, 4096), ("sphere", 200000, 40),
    ("square", 300000, 16),
])
def test_gpu_tree_matches_host(dist, n, leaf):
    _same_tree(host.generate_points(dist, n, 29), leaf)


@pytest.mark.parametrize("n,leaf,sigma", [(20000, 40, 0.02), (200000, 64, 0.01), (50000, 8, 0.05)])
def test_gpu_tree_clustered_balance_replay(n, leaf, sigma):
    # clustered input forces order-dependent 2:1 splits (the host replay path)
    d = _same_tree(_gaussian(n, 3, sigma), leaf)
    assert d.scalars["depth"] >= 5


def test_gpu_tree_degenerate_inputs():
    # collinear, coplanar and grid points (ties on split planes)
    x = np.linspace(0, 1, 4097)
    _same_tree(np.stack([x, np.zeros_like(x), np.zeros_like(x)], 1), 8)
    g = np.stack(np.meshgrid(np.arange(32.0), np.arange(32.0), indexing="ij"), -1).reshape(-1, 2)
    _same_tree(g, 4)
    _same_tree(np.concatenate([g, np.zeros((len(g), 1))], 1) * -3.5, 16)


@requires_ref
@pytest.mark.parametrize("dist,n,leaf", [("cube", 50000, 64), ("sphere", 40000, 30),
                                         ("annulus", 20000, 16)])
def test_gpu_tree_bit_identical_to_reference(dist, n, leaf):
    pts = po.generate_points(dist, n, 5)
    mine = host.HostPlan.build_tree_gpu(pts, leaf).descriptor()
    ref = po.RefPipeline.build(0 if pts.shape[1] == 2 else 1, pts, leaf, 1e-6).descriptor()
    for k in TREE_KEYS:
        assert np.array_equal(mine.arrays[k], ref.arrays[k]), k


def test_gpu_tree_errors():
    pts = host.generate_points("cube", 1000, 1)
    pts[7] = pts[942]
    with pytest.raises(api.DuplicatePointError):
        host.HostPlan.build_tree_gpu(pts, 10)
    with pytest.raises(api.DuplicatePointError):   # duplicates reported before depth
        host.HostPlan.build_tree_gpu(pts, 1)
    with pytest.raises(host.DepthExceededError):
        host.HostPlan.build_tree_gpu(np.array([[0.0, 0.0], [1e-300, 0.0], [1.0, 1.0]]), 1)
    bad = host.generate_points("cube", 50, 1)
    with pytest.raises(ValueError):
        host.HostPlan.build_tree_gpu(bad, 0)
    bad[3, 1] = np.nan
    with pytest.raises(ValueError):
        host.HostPlan.build_tree_gpu(bad, 10)


def test_gpu_tree_feeds_the_apply():
    n = 40000
    pts = host.generate_points("sphere", n, 2)
    hg = host.HostPlan.build_gpu(1, pts, 64, 1e-6, tree="gpu")
    hh = host.HostPlan.build_gpu(1, pts, 64, 1e-6, tree="host")
    q = host.generate_charges(n, 3)
    ug = api.fmm_apply(api.GpuPlan.from_host(hg), q)
    uh = api.fmm_apply(api.GpuPlan.from_host(hh), q)
    assert np.array_equal(ug, uh)


@pytest.mark.parametrize("dist,n,leaf", [("cube", 10_000_000, 128), ("sphere", 3_000_000, 128)])
def test_gpu_tree_matches_host_at_scale(dist, n, leaf):
    # the headline geometry and a large adaptive one (balance replay on the host)
    _same_tree(host.generate_points(dist, n, 1), leaf)

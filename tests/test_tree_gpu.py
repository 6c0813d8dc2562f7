"""GPU tree and neighbor lists: bit-identical to the
unmodified reference build_tree + build_neighbor_lists (oracle/_ref), as
test_tree.cpp:168-200 pins the reference's own tree, box geometry included;
error behaviour as tree.cpp:148-186."""
import numpy as np
import pytest

from conftest import gaussian_points, requires_ref
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
    r = po.RefPipeline.build_tree(pts, leaf)
    dg, dr = g.descriptor(), r.descriptor()
    for k in TREE_KEYS:
        assert np.array_equal(dg.arrays[k], dr.arrays[k]), k
    assert dg.scalars["depth"] == dr.scalars["depth"]
    cg, hg = _geometry(g)
    cr, hr = r.box_geometry()
    assert np.array_equal(cg, cr) and np.array_equal(hg, hr)
    r.close()
    return dg


@pytest.mark.parametrize("dist,n,leaf", [
    ("square", 4000, 20), ("annulus", 8000, 50), ("cube", 5000, 60), ("sphere", 5000, 60),
    ("sphere", 30000, 30), ("cube", 60000, 128), ("annulus", 3000, 1), ("cube", 7, 1),
    ("cube", 1, 1), ("square", 100, 1000), ("cube", 5000, 4096), ("sphere", 200000, 40),
    ("square", 300000, 16), ("cube", 50000, 64), ("sphere", 40000, 30), ("annulus", 20000, 16),
])
@requires_ref
def test_gpu_tree_matches_reference(dist, n, leaf):
    _same_tree(host.generate_points(dist, n, 29), leaf)


@pytest.mark.parametrize("n,leaf,sigma", [(20000, 40, 0.02), (200000, 64, 0.01), (50000, 8, 0.05)])
@requires_ref
def test_gpu_tree_clustered_balance_replay(n, leaf, sigma):
    # clustered input forces order-dependent 2:1 splits (the host replay path)
    d = _same_tree(gaussian_points(n, 3, sigma), leaf)
    assert d.scalars["depth"] >= 5


@requires_ref
def test_gpu_tree_degenerate_inputs():
    # collinear, coplanar and grid points (ties on split planes)
    x = np.linspace(0, 1, 4097)
    _same_tree(np.stack([x, np.zeros_like(x), np.zeros_like(x)], 1), 8)
    g = np.stack(np.meshgrid(np.arange(32.0), np.arange(32.0), indexing="ij"), -1).reshape(-1, 2)
    _same_tree(g, 4)
    _same_tree(np.concatenate([g, np.zeros((len(g), 1))], 1) * -3.5, 16)


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


@pytest.mark.parametrize("dist,n,leaf", [("cube", 10_000_000, 128), ("sphere", 3_000_000, 128)])
@requires_ref
def test_gpu_tree_matches_reference_at_scale(dist, n, leaf):
    # the headline geometry and a large adaptive one (balance replay on the host)
    _same_tree(host.generate_points(dist, n, 1), leaf)

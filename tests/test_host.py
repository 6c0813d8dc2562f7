"""CPU: the host side of the product that is not on the device.

* the benchmark's synthetic inputs are bit-identical to the reference
  generators (bench.cpp:102-161), so the CPU oracle and the GPU see the same
  points and charges;
* the clustered Gaussian of config 3(b) (no reference generator) is
  deterministic and clustered as specified;
* the host descriptor container (include/sfmm_host.h) reproduces a reference
  descriptor it is given (tree adopted, skeletons set) field for field.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import requires_ref
from oracle import pyoracle as po
from paper_2310_16668_b200 import _abi, host


@requires_ref
@pytest.mark.parametrize("dist", ["square", "annulus", "cube", "sphere"])
def test_generators_bit_identical(dist):
    assert np.array_equal(host.generate_points(dist, 5001, 11), po.generate_points(dist, 5001, 11))
    assert np.array_equal(host.generate_charges(5001, 12), po.generate_charges(5001, 12))
    assert np.array_equal(host.generate_charges_complex(5001, 13),
                          po.generate_charges_complex(5001, 13))


def test_gaussian_generator():
    a = host.generate_points("gaussian", 40000, 1)
    b = host.generate_points("gaussian", 40000, 1)
    assert np.array_equal(a, b) and a.shape == (40000, 3)
    assert not np.array_equal(a, host.generate_points("gaussian", 40000, 2))
    # 16 clusters of width 0.02: most points lie within 0.1 of one of 16 centres
    from scipy.cluster.vq import kmeans2
    cent, lab = kmeans2(a, 16, seed=3, minit="++")
    d = np.linalg.norm(a - cent[lab], axis=1)
    assert np.median(d) < 0.06


@requires_ref
@pytest.mark.parametrize("kernel,dist", [(0, "annulus"), (1, "sphere"), (3, "cube")])
def test_descriptor_container_round_trip(kernel, dist):
    """adopt a reference tree, set reference skeletons: the container's
    descriptor equals the reference's field for field."""
    pts = po.generate_points(dist, 3000, 5)
    rp = po.RefPipeline.build(kernel, pts, 40, 1e-6, 2.0)
    ref = rp.descriptor()
    c, h = rp.box_geometry()
    a = ref.arrays
    nb = ref.scalars["n_boxes"]
    # tree arrays in the sfmm_tree_arrays layout (child/morton/cell are not
    # part of the descriptor and are not compared)
    child = np.full(8 * nb, -1, np.int32)
    zeros64 = np.zeros(nb, np.uint64)
    cell = np.zeros(3 * nb, np.int64)
    ta = _abi.TreeArrays()
    keep = [child, zeros64, cell, c, h]
    ta.dim, ta.depth, ta.leaf_cap, ta.n_boxes = ref.scalars["dim"], ref.scalars["depth"], 40, nb
    ta.n_points = ref.n_points
    for f, arr in [("perm", a["perm"]), ("pts", a["pts"]), ("level_begin", a["level_begin"]),
                   ("box_parent", a["box_parent"]), ("box_child", child),
                   ("box_level", a["box_level"]), ("box_morton", zeros64), ("box_cell", cell),
                   ("box_center", c), ("box_half", h), ("box_begin", a["box_begin"]),
                   ("box_end", a["box_end"]), ("box_leaf", a["box_leaf"]),
                   ("coll_off", a["coll_off"]), ("coll", a["coll"]),
                   ("coarse_off", a["coarse_off"]), ("coarse", a["coarse"]),
                   ("fine_off", a["fine_off"]), ("fine", a["fine"])]:
        arr = np.ascontiguousarray(arr)
        keep.append(arr)
        setattr(ta, f, arr.ctypes.data_as(type(getattr(ta, f))))
    hnd = C.c_void_p()
    host._check(host.host_lib().sfmm_host_adopt_tree(C.byref(ta), C.byref(hnd)))
    hp = host.HostPlan(hnd)
    host._check(host.host_lib().sfmm_host_set_skeletons(hp._h, C.byref(ref.struct), kernel, 2.0,
                                                        0, 0, 0, 0.0))
    mine = hp.descriptor()
    for k in ref.arrays:
        assert np.array_equal(mine.arrays[k], ref.arrays[k]), k
    gc, gh = np.zeros(3 * nb), np.zeros(nb)
    host._check(host.host_lib().sfmm_host_box_geometry(hp._h, gc.ctypes.data, gh.ctypes.data))
    assert np.array_equal(gc, c) and np.array_equal(gh, h)
    hp.close()
    rp.close()

"""Generates the golden parity fixtures in tests/golden/ from the REFERENCE.

Run in the build container (it needs oracle/_ref/libsfmm_ref.so, i.e. the
unmodified reference library compiled from /root/reference by oracle/Makefile):

    python tests/golden/make_golden.py

Each fixture stores the flat plan descriptor produced by the reference's own
precompute (build_tree, build_neighbor_lists, build_skeletons), the charges
(reference generators), the reference fmm_apply result ``u_ref`` with its
ApplyStats, and the reference direct sum ``u_direct`` (oracle.cpp:35-49).
The cases follow /root/reference/proj/tests/test_apply.cpp.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as po  # noqa: E402

# name: (kernel, kappa, dist, n, point seed, charge seed, tol, leaf)
CASES = {
    # test_apply.cpp:108-152 (all kernels x geometries, n=1500, tol 1e-6, leaf 40)
    "l2d_square_1500": (0, 1.0, "square", 1500, 100, 200, 1e-6, 40),
    "l2d_annulus_1500": (0, 1.0, "annulus", 1500, 101, 201, 1e-6, 40),
    "l3d_cube_1500": (1, 1.0, "cube", 1500, 102, 202, 1e-6, 40),
    "l3d_sphere_1500": (1, 1.0, "sphere", 1500, 103, 203, 1e-6, 40),
    "h3d_cube_1500": (3, 2.0, "cube", 1500, 102, 202, 1e-6, 40),
    "h3d_sphere_1500": (3, 2.0, "sphere", 1500, 103, 203, 1e-6, 40),
    # test_apply.cpp:154-162 (tight tolerance)
    "l2d_square_2000_tol1e-8": (0, 1.0, "square", 2000, 77, 78, 1e-8, 40),
    # test_apply.cpp:233-254 (annulus, pair counts, ifs/tfo present)
    "l2d_annulus_2500_pairs": (0, 1.0, "annulus", 2500, 61, 62, 1e-5, 25),
    # test_apply.cpp:86-106 (depth-one tree)
    "l2d_square_500_depth1": (0, 1.0, "square", 500, 13, 13, 1e-6, 200),
    # adaptive 3D with a deeper tree (sphere, tol 1e-8)
    "l3d_sphere_6000_tol1e-8": (1, 1.0, "sphere", 6000, 1, 5, 1e-8, 30),
    # headline geometry at small N (uniform cube, leaf 128 -> depth 3)
    "l3d_cube_6000_leaf64": (1, 1.0, "cube", 6000, 1, 1 ^ po.CHARGE_STREAM, 1e-6, 64),
}


def make(name, case):
    kern, kappa, dist, n, ps, cs, tol, leaf = case
    pts = po.generate_points(dist, n, ps)
    cplx = kern >= 2
    q = (po.generate_charges(n, cs).astype(np.complex128) if cplx
         else po.generate_charges(n, cs))
    rp = po.RefPipeline.build(kern, pts, leaf, tol, kappa)
    desc = rp.descriptor()
    u_ref, st = rp.apply(q, cplx)
    u_dir = po.ref_direct_sum(kern, kappa, pts, q)
    info = rp.info()
    path = os.path.join(HERE, f"{name}.npz")
    desc.save(path, q=q, u_ref=u_ref, u_direct=u_dir, points=pts, tol=np.asarray(tol),
              stats=np.asarray([st["n_ifo_pairs"], st["n_ifs_pairs"], st["n_tfo_pairs"],
                                st["n_level1_pairs"], st["direct_fallback"]], dtype=np.int64),
              info=np.asarray([info[k] for k in ("depth", "n_boxes", "k_max", "proj_scalars",
                                                   "saturated_boxes", "n_leaves")], dtype=np.int64))
    print(f"{name}: depth {info['depth']} boxes {info['n_boxes']} k_max {info['k_max']} "
          f"stats {st} -> {os.path.getsize(path) / 1e3:.0f} kB")


if __name__ == "__main__":
    for name, case in CASES.items():
        make(name, case)

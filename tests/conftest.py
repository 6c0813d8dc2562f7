"""Shared fixtures.  GPU tests carry @pytest.mark.gpu; CPU tests never touch a GPU."""
from __future__ import annotations

import ctypes
import glob
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")


def _cuda_device_count() -> int:
    try:
        lib = ctypes.CDLL("libcuda.so.1")
    except OSError:
        return 0
    if lib.cuInit(0) != 0:
        return 0
    n = ctypes.c_int(0)
    if lib.cuDeviceGetCount(ctypes.byref(n)) != 0:
        return 0
    return n.value


HAVE_GPU = _cuda_device_count() > 0


def pytest_collection_modifyitems(config, items):
    if HAVE_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def ensure_built():
    """Builds the product and checker libraries if they are missing (CPU only)."""
    need = [os.path.join(ROOT, "paper_2310_16668_b200", "lib", "libsfmm_gpu.so"),
            os.path.join(ROOT, "paper_2310_16668_b200", "lib", "libsfmm_host.so"),
            os.path.join(ROOT, "oracle", "_build", "libsfmm_oracle.so")]
    if not all(os.path.exists(p) for p in need):
        subprocess.run(["make", "-C", ROOT, "-j8", "all"], check=True)
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8", "oracle"], check=True)
    ref_src = "/root/reference/proj/src"
    ref_so = os.path.join(ROOT, "oracle", "_ref", "libsfmm_ref.so")
    if not os.path.exists(ref_so) and os.path.isdir(ref_src):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8", "ref"], check=True)


ensure_built()


def golden_files():
    return sorted(glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


def load_golden(path):
    from paper_2310_16668_b200._abi import PlanDescriptor
    desc, extra = PlanDescriptor.load(path)
    return desc, extra


def have_ref() -> bool:
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsfmm_ref.so"))


requires_ref = pytest.mark.skipif(not have_ref(), reason="oracle/_ref (reference build) absent")


def ref_descriptor(kernel, pts, leaf, tol, kappa=1.0, proxy=None):
    """Tree, neighbor lists and skeletons from the UNMODIFIED reference pipeline
    (oracle/_ref: build_tree -> build_neighbor_lists -> build_skeletons), as the
    flat descriptor the GPU plan takes -- the same operators the reference CPU
    apply uses, so parity is measured on identical inputs."""
    from oracle import pyoracle as po
    px = proxy or (0.0, 0, 0)
    rp = po.RefPipeline.build(kernel, np.ascontiguousarray(pts, dtype=np.float64), leaf, tol,
                              kappa, float(px[0]), int(px[1]), int(px[2]))
    try:
        return rp.descriptor()
    finally:
        rp.close()


def gaussian_points(n, seed=1, sigma=0.02, clusters=16):
    """Config 3(b) input: 16 Gaussian clusters (the reference has no generator)."""
    from paper_2310_16668_b200 import host
    if seed == 1 and sigma == 0.02 and clusters == 16:
        return host.generate_points("gaussian", n, 1)
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.1, 0.9, size=(clusters, 3))
    return centres[rng.integers(0, clusters, n)] + sigma * rng.standard_normal((n, 3))


def rel_l2(u, ref) -> float:
    u = np.asarray(u)
    ref = np.asarray(ref)
    den = np.linalg.norm(ref.ravel())
    return float(np.linalg.norm((u - ref).ravel()) / (den if den > 0 else 1.0))


def max_rel(u, ref) -> float:
    return float(np.max(np.abs(np.asarray(u) - np.asarray(ref))) / np.max(np.abs(ref)))

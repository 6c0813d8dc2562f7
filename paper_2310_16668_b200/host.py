"""The precompute that feeds the apply, run on the GPU, and its flat descriptor.

Device counterparts of the reference's host API:
    build_tree + build_neighbor_lists  (tree.cpp:148-355)  -> sfmm_gpu_build_tree
    build_skeletons                     (skeleton.cpp:184-260) -> sfmm_gpu_build_skeletons
and the benchmark's synthetic inputs generate_points / generate_charges
(bench.cpp:102-161).  The host library (include/sfmm_host.h) only holds host
copies of the device results as the sfmm_plan_desc consumed by ``api.GpuPlan``.
A C++ caller of the reference keeps the reference's own host precompute and
the drop-in header include/sfmm_gpu.hpp.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _abi
from ._abi import PlanDesc, PlanDescriptor

DIST = {"square": 0, "annulus": 1, "cube": 2, "sphere": 3, "gaussian": 4}
DIST_DIM = {"square": 2, "annulus": 2, "cube": 3, "sphere": 3, "gaussian": 3}
CHARGE_STREAM = 0x9E3779B97F4A7C15  # bench.cpp:27
DEFAULT_LEAF_CAP = {"square": 100, "annulus": 100, "cube": 320, "sphere": 200}  # bench.cpp:92-100
SFMM_EDEPTH = 7


class DepthExceededError(RuntimeError):
    """sfmm::DepthExceededError (common.hpp:25-29)."""


class HostInfo(C.Structure):
    _fields_ = [("depth", C.c_int32), ("n_boxes", C.c_int32), ("n_leaves", C.c_int64),
                ("k_max", C.c_int32), ("saturated_boxes", C.c_int32), ("proj_scalars", C.c_int64),
                ("t_tree", C.c_double), ("t_skel", C.c_double)]


class ProxyConfig(C.Structure):
    _fields_ = [("radius_factor", C.c_double), ("edge_points_2d", C.c_int32),
                ("face_grid_3d", C.c_int32)]


_lib = None


def host_lib() -> C.CDLL:
    global _lib
    if _lib is None:
        path = os.path.join(_abi.LIB_DIR, "libsfmm_host.so")
        if not os.path.exists(path):
            raise _abi.NativeLibraryMissing(f"{path} is missing; run `make`")
        lib = C.CDLL(path)
        vp = C.c_void_p
        lib.sfmm_host_generate_points.argtypes = [C.c_int, C.c_int64, C.c_uint64, vp]
        lib.sfmm_host_generate_charges.argtypes = [C.c_int64, C.c_uint64, vp]
        lib.sfmm_host_generate_charges_complex.argtypes = [C.c_int64, C.c_uint64, vp]
        lib.sfmm_host_desc.argtypes = [vp]
        lib.sfmm_host_desc.restype = C.POINTER(PlanDesc)
        lib.sfmm_host_info_get.argtypes = [vp, C.POINTER(HostInfo)]
        lib.sfmm_host_destroy.argtypes = [vp]
        lib.sfmm_host_destroy.restype = None
        lib.sfmm_host_set_threads.argtypes = [C.c_int]
        lib.sfmm_host_set_threads.restype = None
        lib.sfmm_host_get_threads.restype = C.c_int
        lib.sfmm_host_last_error.restype = C.c_char_p
        lib.sfmm_host_box_geometry.argtypes = [vp, vp, vp]
        lib.sfmm_host_set_skeletons.argtypes = [vp, C.POINTER(PlanDesc), C.c_int, C.c_double,
                                                C.c_int32, C.c_int64, C.c_int32, C.c_double]
        lib.sfmm_host_set_T.argtypes = [vp, vp, C.c_int64]
        lib.sfmm_host_adopt_tree.argtypes = [C.POINTER(_abi.TreeArrays), C.POINTER(vp)]
        _lib = lib
    return _lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    from .api import DuplicatePointError
    msg = host_lib().sfmm_host_last_error().decode()
    if rc == _abi.SFMM_EDUPLICATE:
        raise DuplicatePointError(msg)
    if rc == SFMM_EDEPTH:
        raise DepthExceededError(msg)
    if rc == _abi.SFMM_EINVAL:
        raise ValueError(msg)
    if rc == _abi.SFMM_EUNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == _abi.SFMM_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def generate_points(dist: str, n: int, seed: int) -> np.ndarray:
    out = np.empty((n, DIST_DIM[dist]), dtype=np.float64)
    _check(host_lib().sfmm_host_generate_points(DIST[dist], n, seed, out.ctypes.data))
    return out


def generate_charges(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    _check(host_lib().sfmm_host_generate_charges(n, seed & 0xFFFFFFFFFFFFFFFF, out.ctypes.data))
    return out


def generate_charges_complex(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.complex128)
    _check(host_lib().sfmm_host_generate_charges_complex(n, seed & 0xFFFFFFFFFFFFFFFF,
                                                         out.ctypes.data))
    return out


class HostPlan:
    """Tree + neighbor lists (+ skeletons) built on the host."""

    def __init__(self, handle):
        self._h = handle
        self._skel = None  # device-resident skeleton result (build_gpu(host_T=False))
        self._skel_device = 0

    @classmethod
    def build_gpu(cls, kernel: int, pts: np.ndarray, leaf_cap: int, tol: float,
                  kappa: float = 1.0, proxy: tuple | None = None, device: int = 0,
                  host_T: bool = True, box_mask=None) -> "HostPlan":
        """Tree and neighbor lists (sfmm_gpu_build_tree, bit-identical to the
        reference) and skeletons (sfmm_gpu_build_skeletons), all on the GPU
        (SURVEY.md 8(f) rows 1 and 3).

        host_T=False keeps the interpolation operators on the device only
        (SURVEY.md 8(f) row 2): the descriptor's T is NULL, api.GpuPlan.from_host
        takes T device-to-device, and fetch_T() downloads it when a host copy is
        needed (e.g. for the CPU reference)."""
        hp = cls.build_tree_gpu(pts, leaf_cap, device)
        hp.skeletonize(kernel, tol, kappa, proxy, device, host_T, box_mask)
        return hp

    def skeletonize(self, kernel: int, tol: float, kappa: float = 1.0, proxy: tuple | None = None,
                    device: int = 0, host_T: bool = True, box_mask=None) -> None:
        """Skeletons of this plan's tree on the GPU (sfmm_gpu_build_skeletons).
        box_mask (distributed precompute): only those boxes -- whole subtrees
        -- are skeletonized (sfmm_gpu_build_skeletons_subset); the others stay
        empty, and the device operators are exactly the masked boxes'."""
        from .api import _raise
        hp = self
        d = host_lib().sfmm_host_desc(hp._h).contents
        nb = int(d.n_boxes)
        center = np.zeros(3 * nb)
        half = np.zeros(nb)
        _check(host_lib().sfmm_host_box_geometry(hp._h, center.ctypes.data, half.ctypes.data))
        t = _abi.TreeDesc()
        t.dim, t.n_points, t.n_boxes, t.depth = d.dim, d.n_points, d.n_boxes, d.depth
        for f in ("pts", "level_begin", "box_parent", "box_level", "box_begin", "box_end", "box_leaf"):
            setattr(t, f, getattr(d, f))
        t.box_center = center.ctypes.data_as(C.POINTER(C.c_double))
        t.box_half = half.ctypes.data_as(C.POINTER(C.c_double))
        px = proxy or (0.0, 0, 0)
        res = C.c_void_p()
        lib = _abi.gpu_lib()
        mask = None if box_mask is None else np.ascontiguousarray(box_mask, dtype=np.uint8)
        if mask is not None and mask.size != nb:
            raise ValueError("box_mask must have one entry per box")
        _raise(lib.sfmm_gpu_build_skeletons_subset(
            C.byref(t), kernel, kappa, tol, float(px[0]), int(px[1]), int(px[2]), device,
            None if mask is None else mask.ctypes.data, C.byref(res)))
        keep = False
        try:
            sk = PlanDesc()
            kmax, proj, sat, secs = C.c_int32(), C.c_int64(), C.c_int32(), C.c_double()
            _raise(lib.sfmm_gpu_skel_describe(res, C.byref(sk), 1 if host_T else 0, C.byref(kmax),
                                              C.byref(proj), C.byref(sat), C.byref(secs)))
            _check(host_lib().sfmm_host_set_skeletons(hp._h, C.byref(sk), kernel, kappa, kmax,
                                                      proj, sat, secs))
            keep = not host_T
        finally:
            if keep:
                hp.release_device_skeletons()
                hp._skel, hp._skel_device = res, device
            else:
                lib.sfmm_gpu_skel_destroy(res)

    @property
    def device_skeletons(self):
        """(handle, device) of the device-resident skeletons, or None."""
        return (self._skel, self._skel_device) if self._skel is not None else None

    def device_T(self):
        """(pointer, device, scalars) of the device-resident operators (global
        T_off layout), or None."""
        if self._skel is None:
            return None
        dev, n = C.c_int(), C.c_int64()
        ptr = _abi.gpu_lib().sfmm_gpu_skel_device_T(self._skel, C.byref(dev), C.byref(n))
        return ptr, dev.value, n.value

    def fetch_T(self) -> None:
        """Downloads device-resident interpolation operators into this plan
        (no-op when it already has them)."""
        from .api import _raise
        if self._skel is None or bool(host_lib().sfmm_host_desc(self._h).contents.T):
            return
        lib = _abi.gpu_lib()
        sk = PlanDesc()
        _raise(lib.sfmm_gpu_skel_describe(self._skel, C.byref(sk), 1, None, None, None, None))
        n = C.c_int64()
        lib.sfmm_gpu_skel_device_T(self._skel, None, C.byref(n))
        _check(host_lib().sfmm_host_set_T(self._h, C.cast(sk.T, C.c_void_p), n.value))
        self.release_device_skeletons()  # the result's host copy goes with it

    def release_device_skeletons(self) -> None:
        """Frees the device copy of T held for api.GpuPlan.from_host."""
        if self._skel is not None:
            _abi.gpu_lib().sfmm_gpu_skel_destroy(self._skel)
            self._skel = None

    @classmethod
    def build_tree_gpu(cls, pts: np.ndarray, leaf_cap: int, device: int = 0) -> "HostPlan":
        """Tree and neighbor lists built on the GPU (sfmm_gpu_build_tree,
        SURVEY.md 8(f) row 3), bit-identical to build_tree."""
        from .api import _raise
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        if pts.ndim != 2:
            raise ValueError("build_tree: points must be an (n, dim) array")
        lib = _abi.gpu_lib()
        t = C.c_void_p()
        _raise(lib.sfmm_gpu_build_tree(pts.shape[1], pts.shape[0], pts.ctypes.data, leaf_cap, device,
                                       C.byref(t)))
        try:
            arr = _abi.TreeArrays()
            _raise(lib.sfmm_gpu_tree_arrays(t, C.byref(arr)))
            h = C.c_void_p()
            _check(host_lib().sfmm_host_adopt_tree(C.byref(arr), C.byref(h)))
        finally:
            lib.sfmm_gpu_tree_destroy(t)
        return cls(h)

    def tree_arrays(self) -> _abi.TreeArrays:
        """sfmm_tree_arrays view of this plan's tree (the fields the tree-only
        helpers read: level_begin, box_parent/begin/end/leaf, colleagues);
        valid while this plan is alive."""
        d = self.desc_struct()
        a = _abi.TreeArrays()
        a.dim, a.depth, a.n_boxes, a.n_points = d.dim, d.depth, d.n_boxes, d.n_points
        for f in ("perm", "pts", "level_begin", "box_parent", "box_level", "box_begin", "box_end",
                  "box_leaf", "coll_off", "coll", "coarse_off", "coarse", "fine_off", "fine"):
            setattr(a, f, getattr(d, f))
        return a

    def descriptor(self) -> PlanDescriptor:
        """Owned numpy copy of the flat descriptor."""
        return PlanDescriptor.from_struct(host_lib().sfmm_host_desc(self._h).contents)

    def desc_struct(self) -> PlanDesc:
        """Zero-copy view of the descriptor; valid while this plan is alive."""
        return host_lib().sfmm_host_desc(self._h).contents

    def info(self) -> dict:
        inf = HostInfo()
        _check(host_lib().sfmm_host_info_get(self._h, C.byref(inf)))
        return {k: getattr(inf, k) for k, _ in HostInfo._fields_}

    def close(self) -> None:
        self.release_device_skeletons()
        if self._h is not None:
            host_lib().sfmm_host_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def set_threads(n: int) -> None:
    host_lib().sfmm_host_set_threads(n)


def get_threads() -> int:
    return host_lib().sfmm_host_get_threads()

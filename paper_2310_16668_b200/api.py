"""Python mirror of the reference apply API, running on the sm_100a library.

Reference interface (C++, /root/reference/proj/include/sfmm/apply.hpp):
    struct ApplyStats { n_ifo_pairs, n_ifs_pairs, n_tfo_pairs, n_level1_pairs,
                        direct_fallback };                         apply.hpp:12-18
    template<class K> std::vector<S> fmm_apply(const ApplyPlan<K>&,
                          const std::vector<S>& q, ApplyStats* = nullptr); :91-94
Errors: std::invalid_argument on a charge-count mismatch (apply.cpp:313-314)
-> ValueError; sfmm::DuplicatePointError (a std::domain_error, common.hpp:19-23)
-> DuplicatePointError.

``GpuPlan`` is the device-resident counterpart of ``ApplyPlan<K>``: it is built
once from a flat plan descriptor (tree, neighbor lists, skeletons and
interpolation operators) and keeps everything in HBM.  ``fmm_apply`` takes and
returns potentials in the ORIGINAL point order like the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._abi import PlanDescriptor


class DuplicatePointError(ValueError):
    """sfmm::DuplicatePointError: coincident points with distinct indices."""


class DeviceError(RuntimeError):
    pass


@dataclass
class ApplyStats:
    n_ifo_pairs: int = 0
    n_ifs_pairs: int = 0
    n_tfo_pairs: int = 0
    n_level1_pairs: int = 0
    direct_fallback: bool = False
    ms_total: float = 0.0       # device time of the last apply
    ms_translate: float = 0.0   # device time of the fused translation kernel


def _raise(rc: int) -> None:
    if rc == _abi.SFMM_OK:
        return
    msg = _abi.gpu_lib().sfmm_gpu_last_error().decode()
    if rc == _abi.SFMM_EINVAL:
        raise ValueError(msg)
    if rc == _abi.SFMM_EDUPLICATE:
        raise DuplicatePointError(msg)
    if rc == _abi.SFMM_EUNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == _abi.SFMM_ENOMEM:
        raise MemoryError(msg)
    if rc == _abi.SFMM_EDEPTH:
        from .host import DepthExceededError
        raise DepthExceededError(msg)
    raise DeviceError(msg)


class GpuPlan:
    """Device-resident apply plan (operators uploaded once, resident in HBM)."""

    def __init__(self, desc, device: int = 0, skeletons=None, devices=None):
        """desc: a PlanDescriptor, or a ctypes PlanDesc (e.g. straight from the
        host precompute, without copying its arrays).  skeletons: a device
        skeleton result handle (host.HostPlan.device_skeletons[0]) whose T is
        taken device-to-device instead of desc's T (sfmm_gpu_plan_create_skel).
        devices: several CUDA devices (may repeat) -> one plan sharded over them
        in this process, exchanges by peer copies inside the library
        (sfmm_gpu_plan_create_multi); devices[0] holds q and u."""
        lib = _abi.gpu_lib()
        self.device = device if devices is None else int(devices[0])
        self.devices = None if devices is None else [int(x) for x in devices]
        self._h = None
        if isinstance(desc, PlanDescriptor):
            st = desc.struct
        elif isinstance(desc, _abi.PlanDesc):
            st = desc
        else:
            raise TypeError("GpuPlan: expected a PlanDescriptor or a PlanDesc")
        h = C.c_void_p()
        if self.devices is not None:
            ids = (C.c_int * len(self.devices))(*self.devices)
            if skeletons is not None:
                _raise(lib.sfmm_gpu_plan_create_multi_skel(C.byref(st), skeletons, len(ids), ids,
                                                           C.byref(h)))
            else:
                _raise(lib.sfmm_gpu_plan_create_multi(C.byref(st), len(ids), ids, C.byref(h)))
        elif skeletons is not None:
            _raise(lib.sfmm_gpu_plan_create_skel(C.byref(st), skeletons, device, 1, 0, C.byref(h)))
        else:
            _raise(lib.sfmm_gpu_plan_create(C.byref(st), device, C.byref(h)))
        self._h = h
        self.kernel = int(st.kernel)
        self.n_points = int(st.n_points)
        self.is_complex = self.kernel in (_abi.HELMHOLTZ2D, _abi.HELMHOLTZ3D)
        self.dtype = np.complex128 if self.is_complex else np.float64

    @classmethod
    def from_points(cls, kernel: int, pts, leaf_cap: int, tol: float, kappa: float = 1.0,
                    proxy: tuple | None = None, device: int = 0) -> "GpuPlan":
        """Tree, skeletons and plan in one call, all on the GPU
        (sfmm_gpu_plan_from_points); pts (n, dim) in the original order."""
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        if pts.ndim != 2:
            raise ValueError("from_points: points must be an (n, dim) array")
        px = proxy or (0.0, 0, 0)
        h = C.c_void_p()
        _raise(_abi.gpu_lib().sfmm_gpu_plan_from_points(
            kernel, kappa, pts.shape[1], pts.shape[0], pts.ctypes.data, leaf_cap, tol,
            float(px[0]), int(px[1]), int(px[2]), device, C.byref(h)))
        self = cls.__new__(cls)
        self.device, self._h = device, h
        self.kernel, self.n_points = int(kernel), int(pts.shape[0])
        self.is_complex = self.kernel in (_abi.HELMHOLTZ2D, _abi.HELMHOLTZ3D)
        self.dtype = np.complex128 if self.is_complex else np.float64
        return self

    @classmethod
    def from_host(cls, hp, device: int | None = None, devices=None) -> "GpuPlan":
        """Plan from a host.HostPlan; device-resident skeletons (build_gpu with
        host_T=False) are used in place, so T never crosses PCIe (peer copies
        for a multi-device plan)."""
        ds = hp.device_skeletons
        if devices is not None:
            return cls(hp.desc_struct(), skeletons=None if ds is None else ds[0], devices=devices)
        if ds is not None:
            if device is not None and device != ds[1]:
                raise ValueError("GpuPlan.from_host: skeletons live on another device")
            return cls(hp.desc_struct(), ds[1], skeletons=ds[0])
        return cls(hp.desc_struct(), 0 if device is None else device)

    @property
    def handle(self) -> C.c_void_p:
        if self._h is None:
            raise ValueError("plan has been closed")
        return self._h

    def info(self) -> _abi.PlanInfo:
        inf = _abi.PlanInfo()
        _raise(_abi.gpu_lib().sfmm_gpu_plan_info_get(self.handle, C.byref(inf)))
        return inf

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            _abi.gpu_lib().sfmm_gpu_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def fmm_apply(plan: GpuPlan, q, stats: ApplyStats | None = None,
              out: np.ndarray | None = None) -> np.ndarray:
    """u = A q (apply.cpp:306-337) on the GPU; q, u in original point order.

    q has shape (N,) or (N, nrhs); each column is an independent right-hand side.
    `out` (optional, e.g. a pinned buffer) receives u.
    """
    q = np.asarray(q)
    one = q.ndim == 1
    if q.ndim not in (1, 2) or q.shape[0] != plan.n_points:
        raise ValueError("fmm_apply: charge count does not match the point count")
    qc = np.asfortranarray(q.reshape(plan.n_points, -1), dtype=plan.dtype)
    nrhs = qc.shape[1]
    if out is not None:
        # the C ABI writes n*nrhs contiguous scalars (column-major): a strided
        # view (e.g. big[::2]) would be clobbered between its elements
        if out.dtype != plan.dtype or out.size != qc.size or not out.flags.f_contiguous:
            raise ValueError("fmm_apply: out must be a contiguous (column-major) buffer of "
                             "the result's size and dtype")
        u = out.reshape(plan.n_points, nrhs, order="F")
    else:
        u = np.empty((plan.n_points, nrhs), dtype=plan.dtype, order="F")
    st = _abi.GpuStats()
    _raise(_abi.gpu_lib().sfmm_gpu_apply(plan.handle, qc.ctypes.data, u.ctypes.data, nrhs,
                                         _abi.SFMM_HOST_BUFFERS, C.byref(st)))
    if stats is not None:
        stats.n_ifo_pairs = st.n_ifo_pairs
        stats.n_ifs_pairs = st.n_ifs_pairs
        stats.n_tfo_pairs = st.n_tfo_pairs
        stats.n_level1_pairs = st.n_level1_pairs
        stats.direct_fallback = bool(st.direct_fallback)
        stats.ms_total = st.ms_total
        stats.ms_translate = st.ms_translate
    return u[:, 0] if one else u


def fmm_apply_device(plan: GpuPlan, q_ptr: int, u_ptr: int, nrhs: int = 1, stream: int = 0) -> None:
    """Enqueues u = A q on device buffers (raw pointers) on `stream`; no sync."""
    _raise(_abi.gpu_lib().sfmm_gpu_apply_async(plan.handle, C.c_void_p(q_ptr), C.c_void_p(u_ptr),
                                               nrhs, C.c_void_p(stream or None)))


PHASES = ("gather", "upward", "translate", "downward", "scatter")


def set_timing(plan: GpuPlan, enable: bool = True) -> None:
    """Record per-phase CUDA events in every subsequent apply."""
    _raise(_abi.gpu_lib().sfmm_gpu_set_timing(plan.handle, int(enable)))


def get_timings(plan: GpuPlan, max_applies: int = 256) -> np.ndarray:
    """(n_applies, 5) device ms per phase of the applies recorded since set_timing."""
    ms = np.zeros((max_applies, 5), dtype=np.float32)
    n = C.c_int(0)
    _raise(_abi.gpu_lib().sfmm_gpu_get_timings(plan.handle, ms.ctypes.data, max_applies, C.byref(n)))
    return ms[: n.value].copy()


def fp64_peak_tflops(device: int = 0) -> float:
    """Measured DFMA throughput of the device (TFLOP/s), from the probe library
    (include/sfmm_probe.h; not part of the apply ABI)."""
    v = C.c_double(0)
    rc = _abi.probe_lib().sfmm_probe_fp64_peak(device, C.byref(v))
    if rc != 0:
        raise DeviceError(f"sfmm_probe_fp64_peak failed with code {rc}")
    return v.value


def check_status(plan: GpuPlan) -> None:
    """Syncs and raises DuplicatePointError if an async apply met one."""
    _raise(_abi.gpu_lib().sfmm_gpu_check_status(plan.handle))


def direct_sum_subset(kernel: int, kappa: float, pts: np.ndarray, q: np.ndarray,
                      targets: np.ndarray, device: int = 0) -> np.ndarray:
    """Dense u_i = sum_{j != i} G(x_i,x_j) q_j for the listed targets, on the GPU
    (oracle.cpp:51-71).  pts: (n, dim) in the same order as q."""
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    n, dim = pts.shape
    cplx = kernel in (_abi.HELMHOLTZ2D, _abi.HELMHOLTZ3D)
    qd = np.ascontiguousarray(q, dtype=np.complex128 if cplx else np.float64)
    t = np.ascontiguousarray(targets, dtype=np.int32)
    u = np.empty(t.size, dtype=qd.dtype)
    _raise(_abi.gpu_lib().sfmm_gpu_direct_sum(kernel, float(kappa), dim, n, pts.ctypes.data,
                                              qd.ctypes.data, t.size, t.ctypes.data,
                                              u.ctypes.data, device))
    return u


def max_rel_err(u: np.ndarray, ref: np.ndarray) -> float:
    """max_i |u_i - ref_i| / max_i |ref_i| (oracle.hpp:30-41)."""
    u = np.asarray(u)
    ref = np.asarray(ref)
    if u.shape != ref.shape:
        raise ValueError("max_rel_err: length mismatch")
    den = float(np.max(np.abs(ref))) if ref.size else 0.0
    if den == 0.0:
        raise ArithmeticError("max_rel_err: reference is identically zero")
    return float(np.max(np.abs(u - ref))) / den

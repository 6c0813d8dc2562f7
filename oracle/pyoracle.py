"""TEST INFRASTRUCTURE -- Python handles on the parity checkers.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  It loads

* ``oracle/_ref/libsfmm_ref.so`` -- the UNMODIFIED reference library compiled
  from /root/reference/proj/src by oracle/Makefile, behind the extern "C" shim
  oracle/ref_adapter.cpp;
* ``oracle/_build/libsfmm_oracle.so`` -- the C restatement oracle/sfmm_oracle.c.

Nothing here is part of the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2310_16668_b200._abi import PlanDesc, PlanDescriptor  # noqa: E402

REF_SO = os.path.join(HERE, "_ref", "libsfmm_ref.so")
# the same reference sources and flags plus -march=sapphirerapids (the GPU box
# host's -march=native): the second CPU figure of SURVEY.md 8d
REF_NATIVE_SO = os.path.join(HERE, "_ref", "native", "libsfmm_ref.so")
ORACLE_SO = os.path.join(HERE, "_build", "libsfmm_oracle.so")

DIST = {"square": 0, "annulus": 1, "cube": 2, "sphere": 3}  # bench.hpp:15
DIST_DIM = {"square": 2, "annulus": 2, "cube": 3, "sphere": 3}
CHARGE_STREAM = 0x9E3779B97F4A7C15  # bench.cpp:27
CHECK_STREAM = 0xC2B2AE3D27D4EB4F   # bench.cpp:28

_ref = {}
_orc = None


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def have_oracle() -> bool:
    return os.path.exists(ORACLE_SO)


def have_ref_native() -> bool:
    """The -march build exists and this host CPU can run it (AVX-512 + AMX)."""
    if not os.path.exists(REF_NATIVE_SO):
        return False
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return all(f in flags for f in ("avx512f", "avx512bw", "avx512vl", "amx_tile", "avx512_fp16"))


def ref_lib(native: bool = False) -> C.CDLL:
    if native not in _ref:
        path = REF_NATIVE_SO if native else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle ref)")
        lib = C.CDLL(path)
        vp = C.c_void_p
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_num_threads.restype = C.c_int
        lib.ref_set_threads.argtypes = [C.c_int]
        lib.ref_generate_points.argtypes = [C.c_int, C.c_int64, C.c_uint64, vp]
        lib.ref_generate_charges.argtypes = [C.c_int64, C.c_uint64, vp]
        lib.ref_generate_charges_complex.argtypes = [C.c_int64, C.c_uint64, vp]
        lib.ref_build.argtypes = [C.c_int, C.c_double, C.c_int, C.c_int64, vp, C.c_int, C.c_double,
                                  C.c_double, C.c_int, C.c_int, C.POINTER(vp)]
        lib.ref_build_tree.argtypes = [C.c_int, C.c_int64, vp, C.c_int, C.POINTER(vp)]
        lib.ref_from_desc.argtypes = [C.POINTER(PlanDesc), C.POINTER(vp)]
        lib.ref_desc.argtypes = [vp]
        lib.ref_desc.restype = C.POINTER(PlanDesc)
        lib.ref_box_geometry.argtypes = [vp, vp, vp]
        lib.ref_box_geometry.restype = None
        lib.ref_info.argtypes = [vp, vp]
        lib.ref_info.restype = None
        lib.ref_apply.argtypes = [vp, vp, vp, vp]
        lib.ref_destroy.argtypes = [vp]
        lib.ref_destroy.restype = None
        lib.ref_direct_sum.argtypes = [C.c_int, C.c_double, C.c_int, C.c_int64, vp, vp, C.c_int64,
                                       vp, vp]
        lib.ref_eval_kernel.argtypes = [C.c_int, C.c_double, vp, vp, vp]
        _ref[native] = lib
    return _ref[native]


def oracle_lib() -> C.CDLL:
    global _orc
    if _orc is None:
        if not have_oracle():
            raise FileNotFoundError(f"{ORACLE_SO} not built (make -C oracle oracle)")
        lib = C.CDLL(ORACLE_SO)
        vp = C.c_void_p
        lib.oracle_fmm_apply.argtypes = [C.POINTER(PlanDesc), vp, vp, C.c_int, vp]
        lib.oracle_direct_sum.argtypes = [C.c_int, C.c_double, C.c_int, C.c_int64, vp, vp,
                                          C.c_int64, vp, vp]
        _orc = lib
    return _orc


def _check(rc):
    if rc != 0:
        raise RefError(rc, ref_lib().ref_last_error().decode())


# --- the reference's deterministic generators (bench.cpp:102-161) ----------

def generate_points(dist: str, n: int, seed: int) -> np.ndarray:
    d = DIST_DIM[dist]
    out = np.empty((n, d), dtype=np.float64)
    _check(ref_lib().ref_generate_points(DIST[dist], n, seed, out.ctypes.data))
    return out


def generate_charges(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    _check(ref_lib().ref_generate_charges(n, seed & 0xFFFFFFFFFFFFFFFF, out.ctypes.data))
    return out


def generate_charges_complex(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.complex128)
    _check(ref_lib().ref_generate_charges_complex(n, seed & 0xFFFFFFFFFFFFFFFF, out.ctypes.data))
    return out


class RefPipeline:
    """Reference objects (Tree, NeighborLists, SkeletonSet, ApplyPlan)."""

    def __init__(self, handle, native: bool = False):
        self._h = handle
        self._lib = ref_lib(native)

    @classmethod
    def build(cls, kernel: int, pts: np.ndarray, leaf_cap: int, tol: float, kappa: float = 1.0,
              proxy_radius: float = 0.0, proxy_edge2d: int = 0, proxy_face3d: int = 0,
              native: bool = False):
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        h = C.c_void_p()
        _check(ref_lib(native).ref_build(kernel, kappa, pts.shape[1], pts.shape[0],
                                         pts.ctypes.data, leaf_cap, tol, proxy_radius,
                                         proxy_edge2d, proxy_face3d, C.byref(h)))
        return cls(h, native)

    @classmethod
    def build_tree(cls, pts: np.ndarray, leaf_cap: int):
        """build_tree + build_neighbor_lists only (empty skeleton CSR)."""
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        h = C.c_void_p()
        _check(ref_lib().ref_build_tree(pts.shape[1], pts.shape[0], pts.ctypes.data, leaf_cap,
                                        C.byref(h)))
        return cls(h)

    @classmethod
    def from_desc(cls, desc, native: bool = False):
        """desc: PlanDescriptor or a ctypes PlanDesc (zero-copy view)."""
        st = desc.struct if isinstance(desc, PlanDescriptor) else desc
        h = C.c_void_p()
        _check(ref_lib(native).ref_from_desc(C.byref(st), C.byref(h)))
        return cls(h, native)

    def descriptor(self) -> PlanDescriptor:
        return PlanDescriptor.from_struct(self._lib.ref_desc(self._h).contents)

    def box_geometry(self):
        """(centre (n_boxes*3,), half-width (n_boxes,)) of the reference tree."""
        nb = int(self._lib.ref_desc(self._h).contents.n_boxes)
        c, h = np.zeros(3 * nb), np.zeros(nb)
        self._lib.ref_box_geometry(self._h, c.ctypes.data, h.ctypes.data)
        return c, h

    def info(self) -> dict:
        out = np.zeros(6, dtype=np.int64)
        self._lib.ref_info(self._h, out.ctypes.data)
        keys = ["depth", "n_boxes", "k_max", "proj_scalars", "saturated_boxes", "n_leaves"]
        return dict(zip(keys, (int(v) for v in out)))

    def apply(self, q: np.ndarray, cplx: bool = False):
        q = np.ascontiguousarray(q, dtype=np.complex128 if cplx else np.float64)
        u = np.empty_like(q)
        st = np.zeros(5, dtype=np.int64)
        rc = self._lib.ref_apply(self._h, q.ctypes.data, u.ctypes.data, st.ctypes.data)
        if rc != 0:
            raise RefError(rc, self._lib.ref_last_error().decode())
        return u, dict(zip(["n_ifo_pairs", "n_ifs_pairs", "n_tfo_pairs", "n_level1_pairs",
                            "direct_fallback"], (int(v) for v in st)))

    def close(self):
        if self._h is not None:
            self._lib.ref_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_direct_sum(kernel: int, kappa: float, pts: np.ndarray, q: np.ndarray,
                   targets=None) -> np.ndarray:
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    n, dim = pts.shape
    cplx = kernel >= 2
    q = np.ascontiguousarray(q, dtype=np.complex128 if cplx else np.float64)
    t = np.arange(n, dtype=np.int32) if targets is None else np.ascontiguousarray(targets, np.int32)
    u = np.empty(t.size, dtype=q.dtype)
    _check(ref_lib().ref_direct_sum(kernel, kappa, dim, n, pts.ctypes.data, q.ctypes.data, t.size,
                                    t.ctypes.data, u.ctypes.data))
    return u


def ref_eval_kernel(kernel: int, kappa: float, x, y) -> complex:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    o = np.zeros(2)
    _check(ref_lib().ref_eval_kernel(kernel, kappa, x.ctypes.data, y.ctypes.data, o.ctypes.data))
    return complex(o[0], o[1])


def oracle_apply(desc: PlanDescriptor, q: np.ndarray):
    """The C restatement (sfmm_oracle.c) on a flat descriptor; q (N,) or (N, nrhs)."""
    cplx = desc.is_complex
    q = np.asarray(q)
    one = q.ndim == 1
    qc = np.asfortranarray(q.reshape(desc.n_points, -1), dtype=np.complex128 if cplx else np.float64)
    u = np.empty_like(qc, order="F")
    st = np.zeros(5, dtype=np.int64)
    rc = oracle_lib().oracle_fmm_apply(C.byref(desc.struct), qc.ctypes.data, u.ctypes.data,
                                       qc.shape[1], st.ctypes.data)
    if rc != 0:
        raise RefError(rc, f"oracle_fmm_apply failed with code {rc}")
    stats = dict(zip(["n_ifo_pairs", "n_ifs_pairs", "n_tfo_pairs", "n_level1_pairs",
                      "direct_fallback"], (int(v) for v in st)))
    return (u[:, 0] if one else u), stats


def oracle_direct_sum(kernel: int, kappa: float, pts: np.ndarray, q: np.ndarray, targets=None):
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    n, dim = pts.shape
    cplx = kernel >= 2
    q = np.ascontiguousarray(q, dtype=np.complex128 if cplx else np.float64)
    t = np.arange(n, dtype=np.int32) if targets is None else np.ascontiguousarray(targets, np.int32)
    u = np.empty(t.size, dtype=q.dtype)
    rc = oracle_lib().oracle_direct_sum(kernel, kappa, dim, n, pts.ctypes.data, q.ctypes.data,
                                        t.size, t.ctypes.data, u.ctypes.data)
    if rc != 0:
        raise RefError(rc, f"oracle_direct_sum failed with code {rc}")
    return u


def rel_l2(u, ref) -> float:
    u = np.asarray(u)
    ref = np.asarray(ref)
    den = np.linalg.norm(ref.ravel())
    return float(np.linalg.norm((u - ref).ravel()) / (den if den > 0 else 1.0))

"""ctypes mirror of include/sfmm_gpu.h and the in-tree library loaders.

The product is the C-ABI library ``lib/libsfmm_gpu.so`` (sm_100a CUDA).  This
module only describes its structs and loads it; it never falls back to any CPU
implementation -- a missing library raises ``NativeLibraryMissing``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.environ.get("SFMM_LIB_DIR") or os.path.join(PKG_DIR, "lib")

# kernel ids (sfmm_gpu.h; same order as sfmm::KernelFamily, kernel.hpp:12)
LAPLACE2D, LAPLACE3D, HELMHOLTZ2D, HELMHOLTZ3D = 0, 1, 2, 3
KERNEL_IDS = {"laplace2d": 0, "laplace3d": 1, "helmholtz2d": 2, "helmholtz3d": 3}
KERNEL_DIM = {0: 2, 1: 3, 2: 2, 3: 3}

# return codes
(SFMM_OK, SFMM_EINVAL, SFMM_EDUPLICATE, SFMM_ECUDA, SFMM_ENOMEM, SFMM_ENCCL, SFMM_EUNSUPPORTED,
 SFMM_EDEPTH) = range(8)
SFMM_HOST_BUFFERS, SFMM_DEVICE_BUFFERS = 0, 1

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


class PlanDesc(C.Structure):
    """struct sfmm_plan_desc."""

    _fields_ = [
        ("kernel", C.c_int32),
        ("dim", C.c_int32),
        ("kappa", C.c_double),
        ("n_points", C.c_int64),
        ("n_boxes", C.c_int32),
        ("depth", C.c_int32),
        ("pts", _f64p),
        ("perm", _i32p),
        ("level_begin", _i32p),
        ("box_parent", _i32p),
        ("box_level", _i32p),
        ("box_begin", _i32p),
        ("box_end", _i32p),
        ("box_leaf", _u8p),
        ("box_parent_offset", _i32p),
        ("iv_off", _i64p),
        ("iv", _i32p),
        ("sk_off", _i64p),
        ("skel_pos", _i32p),
        ("rd_off", _i64p),
        ("red_pos", _i32p),
        ("T_off", _i64p),
        ("T", _f64p),
        ("coll_off", _i64p),
        ("coll", _i32p),
        ("coarse_off", _i64p),
        ("coarse", _i32p),
        ("fine_off", _i64p),
        ("fine", _i32p),
    ]


class GpuStats(C.Structure):
    _fields_ = [
        ("n_ifo_pairs", C.c_int64),
        ("n_ifs_pairs", C.c_int64),
        ("n_tfo_pairs", C.c_int64),
        ("n_level1_pairs", C.c_int64),
        ("direct_fallback", C.c_int32),
        ("ms_total", C.c_float),
        ("ms_translate", C.c_float),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("n_points", C.c_int64),
        ("n_boxes", C.c_int32),
        ("depth", C.c_int32),
        ("n_slots", C.c_int64),
        ("n_skel", C.c_int64),
        ("m_proj", C.c_int64),
        ("p_dense", C.c_double),
        ("p_skel", C.c_double),
        ("n_tasks", C.c_int64),
        ("device_bytes", C.c_int64),
        ("n_ifo_pairs", C.c_int64),
        ("n_ifs_pairs", C.c_int64),
        ("n_tfo_pairs", C.c_int64),
        ("n_level1_pairs", C.c_int64),
        ("launches_per_apply", C.c_int32),
        ("k2_grid", C.c_int32),
        ("sym_chain", C.c_int32),
        ("stage_bytes", C.c_int64),
        ("multi_sym", C.c_int32),
        ("merged_tasks", C.c_int32),
        ("multi_stage_bytes", C.c_int64),
    ]


class TreeDesc(C.Structure):
    """struct sfmm_tree_desc (input of the GPU skeletonizer)."""

    _fields_ = [
        ("dim", C.c_int32),
        ("n_points", C.c_int64),
        ("n_boxes", C.c_int32),
        ("depth", C.c_int32),
        ("pts", _f64p),
        ("level_begin", _i32p),
        ("box_parent", _i32p),
        ("box_level", _i32p),
        ("box_begin", _i32p),
        ("box_end", _i32p),
        ("box_leaf", _u8p),
        ("box_center", _f64p),
        ("box_half", _f64p),
    ]


class TreeArrays(C.Structure):
    """struct sfmm_tree_arrays (output of the GPU tree builder)."""

    _fields_ = [
        ("dim", C.c_int32), ("depth", C.c_int32), ("leaf_cap", C.c_int32), ("n_boxes", C.c_int32),
        ("n_points", C.c_int64),
        ("perm", _i32p), ("pts", _f64p), ("level_begin", _i32p), ("box_parent", _i32p),
        ("box_child", _i32p), ("box_level", _i32p), ("box_morton", C.POINTER(C.c_uint64)),
        ("box_cell", _i64p), ("box_center", _f64p), ("box_half", _f64p), ("box_begin", _i32p),
        ("box_end", _i32p), ("box_leaf", _u8p),
        ("coll_off", _i64p), ("coll", _i32p), ("coarse_off", _i64p), ("coarse", _i32p),
        ("fine_off", _i64p), ("fine", _i32p),
        ("seconds", C.c_double),
    ]


# (field, dtype) of every array in the descriptor, in struct order
DESC_ARRAYS = [
    ("pts", np.float64),
    ("perm", np.int32),
    ("level_begin", np.int32),
    ("box_parent", np.int32),
    ("box_level", np.int32),
    ("box_begin", np.int32),
    ("box_end", np.int32),
    ("box_leaf", np.uint8),
    ("box_parent_offset", np.int32),
    ("iv_off", np.int64),
    ("iv", np.int32),
    ("sk_off", np.int64),
    ("skel_pos", np.int32),
    ("rd_off", np.int64),
    ("red_pos", np.int32),
    ("T_off", np.int64),
    ("T", np.float64),
    ("coll_off", np.int64),
    ("coll", np.int32),
    ("coarse_off", np.int64),
    ("coarse", np.int32),
    ("fine_off", np.int64),
    ("fine", np.int32),
]
DESC_SCALARS = ["kernel", "dim", "kappa", "n_points", "n_boxes", "depth"]

_CTYPE = {np.float64: C.c_double, np.int32: C.c_int32, np.int64: C.c_int64, np.uint8: C.c_uint8}


class NativeLibraryMissing(RuntimeError):
    pass


def _array_len(name: str, s: dict, get) -> int:
    nb = int(s["n_boxes"])
    if name == "pts":
        return int(s["n_points"]) * int(s["dim"])
    if name == "perm":
        return int(s["n_points"])
    if name == "level_begin":
        return int(s["depth"]) + 2
    if name.startswith("box_"):
        return nb
    if name.endswith("_off"):
        return nb + 1
    off = {"iv": "iv_off", "skel_pos": "sk_off", "red_pos": "rd_off", "coll": "coll_off",
           "coarse": "coarse_off", "fine": "fine_off", "T": "T_off"}[name]
    n = int(get(off)[nb])
    if name == "T" and int(s["kernel"]) in (HELMHOLTZ2D, HELMHOLTZ3D):
        n *= 2
    return n


class PlanDescriptor:
    """Owns the numpy arrays behind one sfmm_plan_desc.

    Built from a C producer (``from_struct``), from saved arrays
    (``from_arrays`` / ``load``), and handed to the C ABI via ``.struct``.
    """

    def __init__(self, scalars: dict, arrays: dict):
        self.scalars = {k: scalars[k] for k in DESC_SCALARS}
        self.arrays = {}
        for name, dt in DESC_ARRAYS:
            a = np.ascontiguousarray(arrays[name], dtype=dt)
            if a.size == 0:
                a = np.zeros(1, dtype=dt)[:0]
            self.arrays[name] = a
        self._struct = None

    @classmethod
    def from_struct(cls, d: PlanDesc) -> "PlanDescriptor":
        s = {k: getattr(d, k) for k in DESC_SCALARS}
        arrays: dict = {}

        def get(name):
            return arrays[name]

        # offsets first (their lengths do not depend on other arrays)
        order = [n for n, _ in DESC_ARRAYS if n.endswith("_off")] + [
            n for n, _ in DESC_ARRAYS if not n.endswith("_off")]
        dts = dict(DESC_ARRAYS)
        for name in order:
            n = _array_len(name, s, get)
            ptr = getattr(d, name)
            if n == 0 or not ptr:
                arrays[name] = np.zeros(0, dtype=dts[name])
            else:
                arrays[name] = np.ctypeslib.as_array(ptr, shape=(n,)).copy()
        return cls(s, arrays)

    @property
    def struct(self) -> PlanDesc:
        if self._struct is None:
            d = PlanDesc()
            for k in DESC_SCALARS:
                setattr(d, k, self.scalars[k])
            for name, dt in DESC_ARRAYS:
                a = self.arrays[name]
                # an empty array is passed as NULL (e.g. T held on the device only)
                setattr(d, name, a.ctypes.data_as(C.POINTER(_CTYPE[dt])) if a.size else None)
            self._struct = d
        return self._struct

    # convenience views
    @property
    def kernel(self) -> int:
        return int(self.scalars["kernel"])

    @property
    def n_points(self) -> int:
        return int(self.scalars["n_points"])

    @property
    def is_complex(self) -> bool:
        return self.kernel in (HELMHOLTZ2D, HELMHOLTZ3D)

    def save(self, path: str, **extra) -> None:
        np.savez_compressed(path, **{f"s_{k}": np.asarray(v) for k, v in self.scalars.items()},
                            **{f"a_{k}": v for k, v in self.arrays.items()}, **extra)

    @classmethod
    def load(cls, path: str):
        z = np.load(path)
        s = {k: z[f"s_{k}"].item() for k in DESC_SCALARS}
        a = {n: z[f"a_{n}"] for n, _ in DESC_ARRAYS}
        extra = {k: z[k] for k in z.files if not (k.startswith("s_") or k.startswith("a_"))}
        return cls(s, a), extra


_gpu_lib = None


def gpu_lib() -> C.CDLL:
    """Loads lib/libsfmm_gpu.so (the sm_100a product).  Raises if absent."""
    global _gpu_lib
    if _gpu_lib is not None:
        return _gpu_lib
    path = os.path.join(LIB_DIR, "libsfmm_gpu.so")
    if not os.path.exists(path):
        raise NativeLibraryMissing(
            f"{path} is missing; run `make` (or __graft_entry__.build()) -- there is no CPU fallback")
    lib = C.CDLL(path)
    vp = C.c_void_p
    lib.sfmm_gpu_plan_create.argtypes = [C.POINTER(PlanDesc), C.c_int, C.POINTER(vp)]
    lib.sfmm_gpu_plan_create.restype = C.c_int
    lib.sfmm_gpu_apply.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.POINTER(GpuStats)]
    lib.sfmm_gpu_apply.restype = C.c_int
    lib.sfmm_gpu_apply_async.argtypes = [vp, vp, vp, C.c_int, vp]
    lib.sfmm_gpu_apply_async.restype = C.c_int
    lib.sfmm_gpu_check_status.argtypes = [vp]
    lib.sfmm_gpu_check_status.restype = C.c_int
    lib.sfmm_gpu_plan_info_get.argtypes = [vp, C.POINTER(PlanInfo)]
    lib.sfmm_gpu_plan_info_get.restype = C.c_int
    lib.sfmm_gpu_plan_destroy.argtypes = [vp]
    lib.sfmm_gpu_plan_destroy.restype = None
    lib.sfmm_gpu_direct_sum.argtypes = [C.c_int, C.c_double, C.c_int, C.c_int64, vp, vp, C.c_int64,
                                        vp, vp, C.c_int]
    lib.sfmm_gpu_direct_sum.restype = C.c_int
    lib.sfmm_gpu_last_error.argtypes = []
    lib.sfmm_gpu_last_error.restype = C.c_char_p
    lib.sfmm_gpu_version.argtypes = []
    lib.sfmm_gpu_version.restype = C.c_char_p
    lib.sfmm_gpu_set_timing.argtypes = [vp, C.c_int]
    lib.sfmm_gpu_set_timing.restype = C.c_int
    lib.sfmm_gpu_get_timings.argtypes = [vp, vp, C.c_int, C.POINTER(C.c_int)]
    lib.sfmm_gpu_get_timings.restype = C.c_int
    lib.sfmm_gpu_plan_create_sharded.argtypes = [C.POINTER(PlanDesc), C.c_int, C.c_int, C.c_int,
                                                 C.POINTER(vp)]
    lib.sfmm_gpu_plan_create_sharded.restype = C.c_int
    lib.sfmm_gpu_shard_info.argtypes = [vp, vp, vp, vp, vp]
    lib.sfmm_gpu_shard_info.restype = C.c_int
    lib.sfmm_gpu_apply_begin.argtypes = [vp, vp, vp, vp, vp]
    lib.sfmm_gpu_apply_begin.restype = C.c_int
    lib.sfmm_gpu_apply_end.argtypes = [vp, vp, vp, vp, vp]
    lib.sfmm_gpu_apply_end.restype = C.c_int
    lib.sfmm_gpu_shard_info2.argtypes = [vp, vp, vp, C.POINTER(C.c_int)]
    lib.sfmm_gpu_shard_T_runs.argtypes = [C.POINTER(PlanDesc), C.c_int, C.c_int, vp, vp, vp]
    lib.sfmm_gpu_shard_T_runs.restype = C.c_int
    lib.sfmm_gpu_copy_runs.argtypes = [vp, vp, C.c_int64, C.c_int64, vp, C.c_int, vp]
    lib.sfmm_gpu_copy_runs.restype = C.c_int
    lib.sfmm_gpu_plan_create_sharded_T.argtypes = [C.POINTER(PlanDesc), vp, C.c_int, C.c_int,
                                                   C.c_int, C.POINTER(vp)]
    lib.sfmm_gpu_plan_create_sharded_T.restype = C.c_int
    lib.sfmm_gpu_shard_info2.restype = C.c_int
    lib.sfmm_gpu_apply_mid.argtypes = [vp, vp, vp, vp, vp]
    lib.sfmm_gpu_apply_mid.restype = C.c_int
    lib.sfmm_gpu_apply_fin.argtypes = [vp, vp, vp, vp, vp]
    lib.sfmm_gpu_apply_fin.restype = C.c_int
    lib.sfmm_gpu_shard_describe.argtypes = [C.POINTER(PlanDesc), C.c_int, C.c_int, vp, vp, vp, vp,
                                            vp]
    lib.sfmm_gpu_shard_describe.restype = C.c_int
    lib.sfmm_gpu_build_skeletons.argtypes = [C.POINTER(TreeDesc), C.c_int, C.c_double, C.c_double,
                                             C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
    lib.sfmm_gpu_build_skeletons.restype = C.c_int
    lib.sfmm_gpu_skel_fill.argtypes = [vp, C.POINTER(PlanDesc), vp, vp, vp, vp]
    lib.sfmm_gpu_skel_fill.restype = C.c_int
    lib.sfmm_gpu_skel_describe.argtypes = [vp, C.POINTER(PlanDesc), C.c_int, vp, vp, vp, vp]
    lib.sfmm_gpu_skel_describe.restype = C.c_int
    lib.sfmm_gpu_skel_device_T.argtypes = [vp, vp, vp]
    lib.sfmm_gpu_skel_device_T.restype = vp
    lib.sfmm_gpu_plan_create_skel.argtypes = [C.POINTER(PlanDesc), vp, C.c_int, C.c_int, C.c_int,
                                              C.POINTER(vp)]
    lib.sfmm_gpu_plan_create_skel.restype = C.c_int
    lib.sfmm_gpu_build_tree.argtypes = [C.c_int, C.c_int64, vp, C.c_int, C.c_int, C.POINTER(vp)]
    lib.sfmm_gpu_build_tree.restype = C.c_int
    lib.sfmm_gpu_tree_arrays.argtypes = [vp, C.POINTER(TreeArrays)]
    lib.sfmm_gpu_tree_arrays.restype = C.c_int
    lib.sfmm_gpu_tree_destroy.argtypes = [vp]
    lib.sfmm_gpu_tree_destroy.restype = None
    lib.sfmm_gpu_skel_destroy.argtypes = [vp]
    lib.sfmm_gpu_skel_destroy.restype = None
    lib.sfmm_gpu_plan_from_points.argtypes = [C.c_int, C.c_double, C.c_int, C.c_int64, vp, C.c_int,
                                              C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                              C.POINTER(vp)]
    lib.sfmm_gpu_plan_from_points.restype = C.c_int
    lib.sfmm_gpu_plan_create_multi.argtypes = [C.POINTER(PlanDesc), C.c_int, C.POINTER(C.c_int),
                                               C.POINTER(vp)]
    lib.sfmm_gpu_plan_create_multi.restype = C.c_int
    lib.sfmm_gpu_plan_create_multi_skel.argtypes = [C.POINTER(PlanDesc), vp, C.c_int,
                                                    C.POINTER(C.c_int), C.POINTER(vp)]
    lib.sfmm_gpu_plan_create_multi_skel.restype = C.c_int
    lib.sfmm_gpu_nccl_unique_id.argtypes = [vp]
    lib.sfmm_gpu_nccl_unique_id.restype = C.c_int
    lib.sfmm_gpu_plan_attach_nccl.argtypes = [vp, vp, C.c_int, C.c_int]
    lib.sfmm_gpu_plan_attach_nccl.restype = C.c_int
    lib.sfmm_gpu_set_output.argtypes = [vp, C.c_int]
    lib.sfmm_gpu_set_output.restype = C.c_int
    lib.sfmm_gpu_build_skeletons_subset.argtypes = [C.POINTER(TreeDesc), C.c_int, C.c_double,
                                                    C.c_double, C.c_double, C.c_int, C.c_int,
                                                    C.c_int, vp, C.POINTER(vp)]
    lib.sfmm_gpu_build_skeletons_subset.restype = C.c_int
    lib.sfmm_gpu_subtree_owners.argtypes = [C.POINTER(TreeArrays), C.c_int, vp]
    lib.sfmm_gpu_subtree_owners.restype = C.c_int
    lib.sfmm_gpu_plan_create_sharded_owned.argtypes = [C.POINTER(PlanDesc), vp, C.c_int, C.c_int,
                                                       C.c_int, vp, C.POINTER(vp)]
    lib.sfmm_gpu_plan_create_sharded_owned.restype = C.c_int
    _gpu_lib = lib
    return lib


GPU_SYMBOLS = [
    "sfmm_gpu_plan_create", "sfmm_gpu_apply", "sfmm_gpu_apply_async", "sfmm_gpu_check_status",
    "sfmm_gpu_plan_info_get", "sfmm_gpu_plan_destroy", "sfmm_gpu_direct_sum",
    "sfmm_gpu_last_error", "sfmm_gpu_version", "sfmm_gpu_set_timing", "sfmm_gpu_get_timings",
    "sfmm_gpu_plan_create_sharded", "sfmm_gpu_shard_info",
    "sfmm_gpu_apply_begin", "sfmm_gpu_apply_end", "sfmm_gpu_shard_describe",
    "sfmm_gpu_build_skeletons", "sfmm_gpu_skel_fill", "sfmm_gpu_skel_destroy",
    "sfmm_gpu_skel_describe", "sfmm_gpu_skel_device_T",
    "sfmm_gpu_plan_create_skel", "sfmm_gpu_build_tree", "sfmm_gpu_tree_arrays",
    "sfmm_gpu_tree_destroy", "sfmm_gpu_plan_from_points",
    "sfmm_gpu_shard_info2", "sfmm_gpu_apply_mid", "sfmm_gpu_apply_fin",
    "sfmm_gpu_shard_T_runs", "sfmm_gpu_copy_runs", "sfmm_gpu_plan_create_sharded_T",
    "sfmm_gpu_plan_create_multi", "sfmm_gpu_plan_create_multi_skel", "sfmm_gpu_nccl_unique_id",
    "sfmm_gpu_plan_attach_nccl", "sfmm_gpu_set_output", "sfmm_gpu_build_skeletons_subset",
    "sfmm_gpu_subtree_owners", "sfmm_gpu_plan_create_sharded_owned",
]
SFMM_OUTPUT_FULL, SFMM_OUTPUT_OWNED = 0, 1


PROBE_SYMBOLS = ["sfmm_probe_fp64_peak", "sfmm_probe_test_sincos", "sfmm_probe_test_log"]

_probe_lib = None


def probe_lib() -> C.CDLL:
    """Loads lib/libsfmm_probe.so: measurement and test hooks
    (include/sfmm_probe.h), not part of the apply ABI."""
    global _probe_lib
    if _probe_lib is not None:
        return _probe_lib
    path = os.path.join(LIB_DIR, "libsfmm_probe.so")
    if not os.path.exists(path):
        raise NativeLibraryMissing(f"{path} is missing; run `make`")
    lib = C.CDLL(path)
    vp = C.c_void_p
    lib.sfmm_probe_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
    lib.sfmm_probe_fp64_peak.restype = C.c_int
    lib.sfmm_probe_test_sincos.argtypes = [vp, C.c_int64, vp]
    lib.sfmm_probe_test_sincos.restype = C.c_int
    lib.sfmm_probe_test_log.argtypes = [vp, C.c_int64, vp]
    lib.sfmm_probe_test_log.restype = C.c_int
    _probe_lib = lib
    return lib

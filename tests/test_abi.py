"""CPU: the C-ABI libraries load, export every declared symbol, carry sm_100a
code, and validate descriptors before touching a GPU."""
import ctypes as C
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden_files, load_golden, ref_descriptor
from paper_2310_16668_b200 import _abi, api, host

LIB = os.path.join(ROOT, "paper_2310_16668_b200", "lib")


def declared_functions(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sfmm_\w+)\s*\(", text)))


@pytest.mark.parametrize("header,lib", [("sfmm_gpu.h", "libsfmm_gpu.so"),
                                        ("sfmm_host.h", "libsfmm_host.so"),
                                        ("sfmm_probe.h", "libsfmm_probe.so")])
def test_library_exports_every_declared_symbol(header, lib):
    names = declared_functions(header)
    assert names, header
    so = C.CDLL(os.path.join(LIB, lib))
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert set(declared_functions("sfmm_gpu.h")) == set(_abi.GPU_SYMBOLS)
    assert set(declared_functions("sfmm_probe.h")) == set(_abi.PROBE_SYMBOLS)


def test_probe_hooks_are_not_in_the_apply_abi():
    so = C.CDLL(os.path.join(LIB, "libsfmm_gpu.so"))
    for n in _abi.PROBE_SYMBOLS + ["sfmm_gpu_fp64_peak", "sfmm_gpu_test_log", "sfmm_gpu_test_sincos"]:
        assert not hasattr(so, n), n


def test_gpu_library_is_sm100a_code():
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump absent")
    out = subprocess.run([cuobjdump, "--list-elf", os.path.join(LIB, "libsfmm_gpu.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_version_string():
    assert b"sm_100a" in _abi.gpu_lib().sfmm_gpu_version()


def _desc():
    return load_golden(golden_files()[0])[0]


def _create(desc):
    h = C.c_void_p()
    rc = _abi.gpu_lib().sfmm_gpu_plan_create(C.byref(desc.struct), 0, C.byref(h))
    return rc, _abi.gpu_lib().sfmm_gpu_last_error().decode()


@pytest.mark.parametrize("corrupt", ["dim", "perm", "level_begin", "T_off", "skel", "leafrange",
                                     "neighbor"])
def test_plan_create_rejects_bad_descriptors_before_any_cuda_call(corrupt):
    desc = None
    for p in golden_files():
        d, _ = load_golden(p)
        if d.scalars["depth"] >= 2 and d.kernel == 1:
            desc = d
            break
    a = desc.arrays
    if corrupt == "dim":
        desc.scalars["dim"] = 2
    elif corrupt == "perm":
        a["perm"][0] = desc.n_points + 5
    elif corrupt == "level_begin":
        a["level_begin"][-1] += 1
    elif corrupt == "T_off":
        a["T_off"][-1] += 1
    elif corrupt == "skel":
        b = int(np.nonzero(np.diff(a["sk_off"]))[0][-1])
        a["skel_pos"][a["sk_off"][b]] = 10 ** 6
    elif corrupt == "leafrange":
        b = int(np.nonzero(a["box_leaf"])[0][0])
        a["box_end"][b] += 1
    elif corrupt == "neighbor":
        a["coll"][0] = desc.scalars["n_boxes"] + 3
    desc._struct = None
    rc, msg = _create(desc)
    assert rc == _abi.SFMM_EINVAL, (rc, msg)
    assert msg.startswith("sfmm_gpu_plan_create")


def test_helmholtz2d_plan_is_unsupported():
    d = _desc()
    d.scalars["kernel"] = _abi.HELMHOLTZ2D
    d._struct = None
    rc, _ = _create(d)
    assert rc == _abi.SFMM_EUNSUPPORTED


def test_error_mapping_to_python_exceptions():
    d = _desc()
    d.scalars["dim"] = 3 if d.scalars["dim"] == 2 else 2
    d._struct = None
    with pytest.raises(ValueError):
        api.GpuPlan(d)


def test_descriptor_roundtrip_through_npz(tmp_path):
    d = ref_descriptor(1, host.generate_points("cube", 800, 2), 30, 1e-6)
    p = tmp_path / "d.npz"
    d.save(str(p))
    d2, _ = _abi.PlanDescriptor.load(str(p))
    for k in d.arrays:
        assert np.array_equal(d.arrays[k], d2.arrays[k])
    assert d.scalars == d2.scalars


def test_nccl_unique_id_without_gpu():
    # the library loads NCCL at run time (dlopen) for the one-process-per-GPU
    # exchange; making a communicator id needs no device
    from paper_2310_16668_b200 import shard
    uid = shard.nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == shard.NCCL_ID_BYTES and any(uid)

"""Multi-GPU apply with the exchanges inside the C ABI.

sfmm_gpu_plan_create_multi shards one plan over several devices of this
process and exchanges ghosts and column sums with one cudaMemcpyPeerAsync per
peer segment.  Device ids may repeat, so the whole data plane -- per-rank
plans, peer copies, cross-device events, gather of q and scatter of u through
the primary device -- runs on the single B200 of a gpurun box as N virtual
ranks.  The reference's contract (apply.hpp:88-94: u in the original order,
deterministic) is checked against the single-GPU plan and the reference CPU
apply on the same operators.
"""
import numpy as np
import pytest

from conftest import ref_descriptor, rel_l2, requires_ref
from oracle import pyoracle as po
from paper_2310_16668_b200 import _abi, api, host, shard

pytestmark = pytest.mark.gpu

PARITY = 1e-12


def _case(name):
    kern, dist, kappa, n, leaf, tol = {
        "l3d_cube": (1, "cube", 1.0, 60000, 64, 1e-6),
        "l3d_sphere": (1, "sphere", 1.0, 60000, 64, 1e-8),
        "l3d_gaussian": (1, "gaussian", 1.0, 60000, 64, 1e-6),
        "l2d_square": (0, "square", 1.0, 40000, 64, 1e-6),
        "h3d_cube": (3, "cube", 10.0, 20000, 64, 1e-6),
    }[name]
    pts = host.generate_points(dist, n, 1)
    d = ref_descriptor(kern, pts, leaf, tol, kappa)
    gen = host.generate_charges_complex if kern == 3 else host.generate_charges
    return d, gen(n, 5), kern


@requires_ref
@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0], [0, 0, 0, 0], [0] * 8])
@pytest.mark.parametrize("case", ["l3d_cube", "l3d_sphere", "l3d_gaussian", "l2d_square",
                                  "h3d_cube"])
def test_multi_device_plan_matches_reference(devices, case):
    d, q, kern = _case(case)
    u_single = api.fmm_apply(api.GpuPlan(d), q)
    st = api.ApplyStats()
    with api.GpuPlan(d, devices=devices) as plan:
        u = api.fmm_apply(plan, q, st)
        # repeated applies are bit-identical (determinism, test_apply.cpp:206-231)
        assert np.array_equal(api.fmm_apply(plan, q), u)
    rp = po.RefPipeline.from_desc(d)
    u_ref, st_ref = rp.apply(q, kern == 3)
    rp.close()
    assert rel_l2(u, u_ref) <= PARITY
    assert rel_l2(u, u_single) <= PARITY
    assert (st.n_ifo_pairs, st.n_ifs_pairs, st.n_tfo_pairs, st.n_level1_pairs) == (
        st_ref["n_ifo_pairs"], st_ref["n_ifs_pairs"], st_ref["n_tfo_pairs"],
        st_ref["n_level1_pairs"])


def test_multi_device_plan_clustered_uses_level2_cut():
    d, q, _ = _case("l3d_gaussian")
    assert shard.describe(d, 8, 0)["cut_level"] == 2
    u_single = api.fmm_apply(api.GpuPlan(d), q)
    with api.GpuPlan(d, devices=[0] * 8) as plan:
        assert rel_l2(api.fmm_apply(plan, q), u_single) <= PARITY


def test_multi_device_plan_async_and_multi_rhs():
    import torch
    d, q, _ = _case("l3d_cube")
    n = d.n_points
    Q = np.asfortranarray(np.stack([host.generate_charges(n, 40 + r) for r in range(3)], 1))
    with api.GpuPlan(d) as single:
        U_single = api.fmm_apply(single, Q)
    with api.GpuPlan(d, devices=[0, 0, 0, 0]) as plan:
        U = api.fmm_apply(plan, Q)                 # column by column
        assert rel_l2(U, U_single) <= PARITY
        qd = torch.from_numpy(np.ascontiguousarray(Q[:, 0])).cuda()
        ud = torch.empty_like(qd)
        s = torch.cuda.Stream()
        for _ in range(3):                         # phase graphs replayed
            api.fmm_apply_device(plan, qd.data_ptr(), ud.data_ptr(), 1, s.cuda_stream)
        api.check_status(plan)
        assert np.array_equal(ud.cpu().numpy(), U[:, 0])
        inf = plan.info()
        assert inf.launches_per_apply > 0 and inf.device_bytes > 0


def test_multi_device_plan_from_device_skeletons():
    # GPU precompute: the operators stay on the device and every rank takes its
    # owned runs device-to-device (sfmm_gpu_plan_create_multi_skel)
    n = 40000
    pts = host.generate_points("cube", n, 2)
    hp = host.HostPlan.build_gpu(1, pts, 64, 1e-6, host_T=False)
    q = host.generate_charges(n, 6)
    with api.GpuPlan.from_host(hp) as single:
        u_single = api.fmm_apply(single, q)
    with api.GpuPlan.from_host(hp, devices=[0, 0, 0]) as plan:
        assert rel_l2(api.fmm_apply(plan, q), u_single) <= PARITY
    hp.close()


def test_multi_device_plan_depth0_and_errors():
    pts = host.generate_points("cube", 60, 3)
    d = ref_descriptor(1, pts, 100, 1e-6)            # depth 0: dense fallback on rank 0
    q = host.generate_charges(60, 4)
    with api.GpuPlan(d, devices=[0, 0]) as plan:
        assert np.array_equal(api.fmm_apply(plan, q), api.fmm_apply(api.GpuPlan(d), q))
    with pytest.raises((api.DeviceError, ValueError)):
        api.GpuPlan(d, devices=[0, 99])               # no such device
    # the caller-driven exchange entry points refuse a self-exchanging plan
    import ctypes as C
    d2, _, _ = _case("l3d_cube")
    with api.GpuPlan(d2, devices=[0, 0]) as plan:
        rc = _abi.gpu_lib().sfmm_gpu_apply_begin(plan.handle, C.c_void_p(1), None, None, None)
        assert rc == _abi.SFMM_EINVAL


def test_multi_device_duplicate_points_reported():
    # apply.cpp:31-33 through the sharded path: a valid plan, then one point
    # moved onto another inside the same leaf (the leaf lives on some rank)
    pts = host.generate_points("cube", 20000, 7)
    d = ref_descriptor(1, pts, 40, 1e-6)
    a = d.arrays
    leaves = np.nonzero(a["box_leaf"] & (a["box_end"] - a["box_begin"] >= 2))[0]
    leaf = int(leaves[len(leaves) // 2])
    t0, t1 = a["box_begin"][leaf], a["box_begin"][leaf] + 1
    P = a["pts"].reshape(-1, 3)
    P[t1] = P[t0]
    d._struct = None
    with api.GpuPlan(d, devices=[0, 0, 0, 0]) as plan:
        with pytest.raises(api.DuplicatePointError):
            api.fmm_apply(plan, host.generate_charges(20000, 1))


def test_nccl_rank_plan_single_rank():
    """The one-process-per-GPU transport on the one GPU a gpurun box has: a
    1-rank NCCL communicator exercises the run-time NCCL load, the
    communicator set-up and the collective apply (grouped send/recv with no
    peers, the in-place all-reduce of the full result, the owned-only output)
    -- everything but the peer traffic."""
    import torch
    d, q, _ = _case("l3d_sphere")
    u_single = api.fmm_apply(api.GpuPlan(d), q)
    plan = shard.ShardedPlan(d, 1, 0)
    plan.attach_nccl(shard.nccl_unique_id())
    qd = torch.from_numpy(q).cuda()
    ud = torch.zeros_like(qd)
    s = torch.cuda.Stream()
    plan.set_output(owned_only=True)
    plan.apply(qd, ud, s.cuda_stream)
    s.synchronize()
    assert rel_l2(ud.cpu().numpy(), u_single) <= PARITY
    plan.set_output(owned_only=False)
    out = np.empty_like(q)
    plan.apply_host(np.ascontiguousarray(q), out)
    assert rel_l2(out, u_single) <= PARITY
    plan.close()


def test_bench_sharded_path_one_rank_nccl_in_library(tmp_path):
    """bench.py's multi-rank path (torchrun, NCCL process group, operator blobs,
    the exchange inside the library) end to end with one rank."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "bench.py"), "--force-sharded", "--steps", "2", "--warmup", "3",
           "--points", "3e5", "--check-targets", "100"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["exchange_in_library"] is True, line["parallelism"]
    assert line["relerr_vs_single_gpu"] <= 1e-12
    assert line["value"] > 0 and line["e2e"]["value"] > 0


@pytest.mark.parametrize("case", ["l3d_cube", "l3d_sphere", "h3d_cube"])
def test_multi_device_overlapped_exchange(case, monkeypatch):
    """SFMM_SHARD_OVERLAP=1: each rank's interior tasks (no ghost source) run
    while the ghost exchange is in flight on the rank's exchange stream (peer
    copies), the boundary tasks after it; same result as the plain plan,
    bit-identical repeats."""
    d, q, _ = _case(case)
    with api.GpuPlan(d, devices=[0, 0, 0, 0]) as plan:
        u0 = api.fmm_apply(plan, q)
    monkeypatch.setenv("SFMM_SHARD_OVERLAP", "1")
    with api.GpuPlan(d, devices=[0, 0, 0, 0]) as plan:
        u = api.fmm_apply(plan, q)
        assert np.array_equal(api.fmm_apply(plan, q), u)
    assert rel_l2(u, u0) <= 1e-13


@pytest.mark.parametrize("case", ["l3d_cube", "h3d_cube"])
@pytest.mark.parametrize("overlap", ["0", "1"])
def test_multi_device_merged_tile_tasks(case, overlap, monkeypatch):
    """The merged-task staging layout on rank plans (cross-rank colleague pairs'
    column sums packed from one staged vector per pair; interior / boundary
    task parts with the overlap): same result as the per-tile rank plans."""
    d, q, _ = _case(case)
    monkeypatch.setenv("SFMM_SHARD_OVERLAP", overlap)
    with api.GpuPlan(d, devices=[0, 0, 0, 0]) as plan:
        u0 = api.fmm_apply(plan, q)
    monkeypatch.setenv("SFMM_MERGE_TILES", "1")
    monkeypatch.setenv("SFMM_MERGE_SHARE", "1e9")
    with api.GpuPlan(d, devices=[0, 0, 0, 0]) as plan:
        assert plan.info().merged_tasks > 0
        u = api.fmm_apply(plan, q)
        assert np.array_equal(api.fmm_apply(plan, q), u)
    assert rel_l2(u, u0) <= 1e-13

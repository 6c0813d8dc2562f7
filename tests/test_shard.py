"""Multi-GPU sharding.

CPU: the shard layout every rank derives independently is consistent
(ownership, owned-point partition, matching ghost send/receive lists), checked
in one process for 2/4/8 ranks and across a real world_size-2 gloo group.
GPU: the sharded apply, run as N virtual ranks on the single available GPU
(sequential, exchange by device copies), reproduces the single-plan result.
"""
import os
import socket

import numpy as np
import pytest

from conftest import max_rel, ref_descriptor, rel_l2
from paper_2310_16668_b200 import api, host, shard


def _desc(dist="cube", n=20000, leaf=64, kernel=1, tol=1e-6, kappa=1.0, seed=1):
    pts = host.generate_points(dist, n, seed)
    return ref_descriptor(kernel, pts, leaf, tol, kappa), pts


@pytest.mark.parametrize("n_ranks", [1, 2, 4, 8])
@pytest.mark.parametrize("dist", ["cube", "sphere"])
def test_shard_layout_consistent(n_ranks, dist):
    d, _ = _desc(dist=dist)
    infos = [shard.describe(d, n_ranks, r) for r in range(n_ranks)]
    owner = infos[0]["owner"]
    for inf in infos:
        assert np.array_equal(inf["owner"], owner)  # every rank derives the same split
    cut = infos[0]["cut_level"]
    lvl = d.arrays["box_level"]
    shared = owner == -1
    assert set(np.unique(owner[~shared])) == set(range(n_ranks))
    # shared boxes: the internal level-1 boxes of a level-2 cut, nothing else
    assert np.all(lvl[shared] == 1) and (cut == 2 or not shared.any())
    assert not np.any(d.arrays["box_leaf"][shared].astype(bool))
    # owned points partition the point set
    pts = np.concatenate([inf["owned_points"] for inf in infos])
    assert np.array_equal(np.sort(pts), np.arange(d.n_points))
    # what p sends to q is exactly what q expects from p, element by element
    for p in range(n_ranks):
        s_off = np.concatenate([[0], np.cumsum(infos[p]["send_counts"])])
        for q in range(n_ranks):
            r_off = np.concatenate([[0], np.cumsum(infos[q]["recv_counts"])])
            sent = infos[p]["pack_idx"][s_off[q]:s_off[q + 1]]
            got = infos[q]["unpack_idx"][r_off[p]:r_off[p + 1]]
            assert np.array_equal(sent, got), (p, q)
            if p == q:
                assert sent.size == 0
    # second exchange (cross-rank colleague pairs evaluated on one side)
    for p in range(n_ranks):
        assert infos[p]["send2_counts"][p] == 0 and infos[p]["recv2_counts"][p] == 0
        for q in range(n_ranks):
            assert infos[p]["send2_counts"][q] == infos[q]["recv2_counts"][p], (p, q)
    if n_ranks > 1:
        assert sum(int(inf["send2_counts"].sum()) for inf in infos) > 0
    # ghosts are never owned by the receiver
    a = d.arrays
    n_slots = int(a["iv_off"][-1])
    for q, inf in enumerate(infos):
        idx = inf["unpack_idx"]
        slot_idx = idx[idx < n_slots]
        box_of_slot = np.searchsorted(a["iv_off"], slot_idx, side="right") - 1
        assert np.all(owner[box_of_slot] != q)


def _shuffled_colleagues(d, seed=7):
    """The same descriptor with every colleague list in a random order."""
    from paper_2310_16668_b200._abi import PlanDescriptor
    a = {k: v.copy() for k, v in d.arrays.items()}
    rng = np.random.default_rng(seed)
    off, coll = a["coll_off"], a["coll"]
    for b in range(len(off) - 1):
        seg = coll[off[b]:off[b + 1]]
        coll[off[b]:off[b + 1]] = seg[rng.permutation(seg.size)]
    return PlanDescriptor(d.scalars, a)


def test_unsorted_colleague_lists_disable_the_fold():
    # the one-sided cross-rank pairs look pairs up in sorted colleague lists;
    # a descriptor with unsorted lists must fall back to two-sided pairs
    d, _ = _desc()
    assert sum(int(shard.describe(d, 4, r)["send2_counts"].sum()) for r in range(4)) > 0
    ds = _shuffled_colleagues(d)
    infos = [shard.describe(ds, 4, r) for r in range(4)]
    assert all(int(i["send2_counts"].sum()) == 0 and int(i["recv2_counts"].sum()) == 0 for i in infos)


@pytest.mark.parametrize("dist,n_ranks", [("cube", 4), ("cube", 8), ("gaussian", 8)])
def test_subtrees_are_owned_whole(dist, n_ranks):
    d, _ = _desc(dist=dist, n=40000)
    inf = shard.describe(d, n_ranks, 0)
    owner, cut = inf["owner"], inf["cut_level"]
    parent = d.arrays["box_parent"]
    lvl = d.arrays["box_level"]
    for b in range(1, d.scalars["n_boxes"]):
        if lvl[b] > cut:
            assert owner[b] == owner[parent[b]]
    if cut == 2:  # every level-2 subtree has one owner; the level-1 boxes above them are shared
        assert np.all(owner[lvl == 2] >= 0)


def test_clustered_input_uses_the_level2_cut():
    # 16-cluster Gaussian (config 3b geometry): level-1 subtrees are far apart
    # in cost (max/mean 2.21 at 8 ranks); the plan cuts at level 2
    d, _ = _desc(dist="gaussian", n=60000, tol=1e-8)
    infos = [shard.describe(d, 8, r) for r in range(8)]
    assert infos[0]["cut_level"] == 2
    owner = infos[0]["owner"]
    lvl = d.arrays["box_level"]
    assert np.all(owner[(lvl == 1) & ~d.arrays["box_leaf"].astype(bool)] == -1)
    assert all(i["n_owned_points"] > 0 for i in infos)
    # every rank receives the shared level-1 slots filled by the other ranks
    iv = d.arrays["iv_off"]
    for r, inf in enumerate(infos):
        idx = inf["unpack_idx"]
        box_of = np.searchsorted(iv, idx[idx < iv[-1]], side="right") - 1
        got_shared = np.unique(box_of[owner[box_of] == -1])
        kids = [c for c in np.nonzero(lvl == 2)[0] if owner[c] != r]
        assert set(got_shared) == set(d.arrays["box_parent"][kids])


def _lopsided(seed=3):
    """A depth-2 tree: two octants split into level-2 boxes, the sparse others
    stay level-1 leaves (2:1 balance allows leaves only next to level <= 2)."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.0, 0.5, (300, 3))
    b = rng.uniform(0.5, 1.0, (300, 3))
    few = rng.uniform(0.0, 1.0, (200, 3))
    return np.ascontiguousarray(np.concatenate([a, b, few]))


def test_level1_leaves_are_units():
    pts = _lopsided()
    d = ref_descriptor(1, pts, 64, 1e-6, 1.0)
    leaf1 = np.nonzero((d.arrays["box_level"] == 1) & d.arrays["box_leaf"].astype(bool))[0]
    assert leaf1.size > 0
    infos = [shard.describe(d, 8, r) for r in range(8)]
    assert infos[0]["cut_level"] == 2
    owner = infos[0]["owner"]
    assert np.all(owner[leaf1] >= 0)  # owned, not shared
    pts_owned = np.sort(np.concatenate([i["owned_points"] for i in infos]))
    assert np.array_equal(pts_owned, np.arange(d.n_points))
    for p in range(8):
        for q in range(8):
            assert infos[p]["send_counts"][q] == infos[q]["recv_counts"][p]
            assert infos[p]["send2_counts"][q] == infos[q]["recv2_counts"][p]


def test_too_many_ranks_is_unsupported():
    d, _ = _desc(dist="square", kernel=0, n=5000, leaf=32)  # 2D: 4 level-1, <= 16 level-2 boxes
    shard.describe(d, 8, 0)  # level-2 cut
    with pytest.raises(NotImplementedError):
        shard.describe(d, 64, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, _ = _desc(dist="sphere", n=12000, leaf=40)
        inf = shard.describe(d, world, rank)
        # counts: what I send to p must equal what p receives from me
        send = torch.tensor(inf["send_counts"], dtype=torch.int64)
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send)
        ok = bool(torch.equal(recv, torch.tensor(inf["recv_counts"], dtype=torch.int64)))
        # payload: ship the packed element indices, compare with my unpack list
        payload = torch.tensor(inf["pack_idx"], dtype=torch.int64)
        got = torch.empty(int(inf["recv_counts"].sum()), dtype=torch.int64)
        dist.all_to_all_single(got, payload, output_split_sizes=inf["recv_counts"].tolist(),
                               input_split_sizes=inf["send_counts"].tolist())
        ok = ok and bool(np.array_equal(got.numpy(), inf["unpack_idx"]))
        # owned points: disjoint union over ranks
        gathered = [None] * world
        dist.all_gather_object(gathered, inf["owned_points"])
        allp = np.sort(np.concatenate(gathered))
        ok = ok and bool(np.array_equal(allp, np.arange(d.n_points)))
        out[rank] = ok
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_plan():
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gloo_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0] and out[1]


# ---------------------------------------------------------------------------
# GPU: sharded apply on one device (virtual ranks)
# ---------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("n_ranks", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("case", ["l3d_cube", "l3d_sphere", "h3d_cube", "l3d_gaussian"])
def test_virtual_ranks_match_single_plan(n_ranks, case):
    import torch
    kern, dist, kappa = {"l3d_cube": (1, "cube", 1.0), "l3d_sphere": (1, "sphere", 1.0),
                         "h3d_cube": (3, "cube", 5.0), "l3d_gaussian": (1, "gaussian", 1.0)}[case]
    n = 30000 if kern == 1 else 12000
    d, pts = _desc(dist=dist, n=n, leaf=64, kernel=kern, kappa=kappa)
    if case == "l3d_gaussian" and n_ranks == 8:  # clustered: level-2 cut, shared level-1 boxes
        assert shard.describe(d, n_ranks, 0)["cut_level"] == 2
    q = host.generate_charges_complex(n, 3) if kern == 3 else host.generate_charges(n, 3)
    u_ref = api.fmm_apply(api.GpuPlan(d), q)
    plans = [shard.ShardedPlan(d, n_ranks, r) for r in range(n_ranks)]
    assert sum(p.n_owned_points for p in plans) == n
    qd = torch.from_numpy(q).cuda()
    ud = torch.zeros_like(qd)
    shard.apply_virtual(plans, qd, ud)
    torch.cuda.synchronize()
    u = ud.cpu().numpy()
    assert rel_l2(u, u_ref) <= 1e-12
    if n_ranks > 1:
        assert any(p.n_ghost_boxes > 0 for p in plans)


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"SFMM_SHARD_XSYM": "0"}, {"SFMM_SHARD_OVERLAP": "1"},
                                 {"SFMM_SHARD_OVERLAP": "1", "SFMM_SHARD_XSYM": "0"}])
def test_virtual_ranks_plan_variants(env, monkeypatch):
    # the one-sided cross-rank pairs (default) against both sides evaluating
    # them, and the overlapped two-launch split; all must match the single plan
    import torch
    n = 30000
    d, pts = _desc(dist="sphere", n=n, leaf=64)
    q = host.generate_charges(n, 3)
    u_ref = api.fmm_apply(api.GpuPlan(d), q)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    plans = [shard.ShardedPlan(d, 4, r) for r in range(4)]
    assert all(p.cross_symmetric == (env.get("SFMM_SHARD_XSYM") != "0") for p in plans)
    qd = torch.from_numpy(q).cuda()
    ud = torch.zeros_like(qd)
    shard.apply_virtual(plans, qd, ud)
    torch.cuda.synchronize()
    assert rel_l2(ud.cpu().numpy(), u_ref) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("kernel,n_ranks", [(1, 4), (1, 8), (3, 3)])
def test_sharded_plans_from_device_operator_blobs(kernel, n_ranks):
    # the descriptor travels without T; each rank's operators are packed from
    # the device-resident skeletons (what rank 0 ships over NCCL at N=1e8)
    import torch
    n = 30000 if kernel == 1 else 12000
    pts = host.generate_points("cube", n, 1)
    hp = host.HostPlan.build_gpu(kernel, pts, 64, 1e-6, 5.0, host_T=False)
    d = hp.desc_struct()
    assert not bool(d.T)
    q = host.generate_charges_complex(n, 3) if kernel == 3 else host.generate_charges(n, 3)
    u_ref = api.fmm_apply(api.GpuPlan.from_host(hp), q)
    ptr, dev, n_scalars = hp.device_T()
    sw = 2 if kernel == 3 else 1
    plans, total = [], 0
    for r in range(n_ranks):
        runs, n_entries = shard.T_runs(d, n_ranks, r)
        assert int(runs[:, 1].sum()) == n_entries
        blob = torch.empty(max(1, n_entries * sw), dtype=torch.float64, device="cuda")
        shard.pack_T(ptr, runs, sw, blob, dev)
        plans.append(shard.ShardedPlan(d, n_ranks, r, T_owned=blob))
        total += n_entries * sw
    assert total <= n_scalars  # shared boxes carry no operators
    qd = torch.from_numpy(q).cuda()
    ud = torch.zeros_like(qd)
    shard.apply_virtual(plans, qd, ud)
    torch.cuda.synchronize()
    assert rel_l2(ud.cpu().numpy(), u_ref) <= 1e-12


@pytest.mark.gpu
def test_unsorted_colleague_lists_same_result():
    import torch
    n = 30000
    d, _ = _desc(n=n, leaf=64)
    ds = _shuffled_colleagues(d)
    q = host.generate_charges(n, 3)
    u_ref = api.fmm_apply(api.GpuPlan(d), q)
    assert rel_l2(api.fmm_apply(api.GpuPlan(ds), q), u_ref) <= 1e-12
    plans = [shard.ShardedPlan(ds, 4, r) for r in range(4)]
    assert not any(p.cross_symmetric for p in plans)
    qd = torch.from_numpy(q).cuda()
    ud = torch.zeros_like(qd)
    shard.apply_virtual(plans, qd, ud)
    torch.cuda.synchronize()
    assert rel_l2(ud.cpu().numpy(), u_ref) <= 1e-12


@pytest.mark.gpu
def test_cross_symmetric_plan_requires_mid_fin():
    import torch
    n = 30000
    d, _ = _desc(n=n, leaf=64)
    plans = [shard.ShardedPlan(d, 2, r) for r in range(2)]
    assert all(p.cross_symmetric for p in plans)
    assert sum(int(p.send2_counts.sum()) for p in plans) > 0
    qd = torch.zeros(n, dtype=torch.float64, device="cuda")
    plans[0].begin(qd, 0, 0)
    with pytest.raises(ValueError, match="apply_mid"):
        plans[0].end(qd, torch.zeros_like(qd), 0)
    torch.cuda.synchronize()


@pytest.mark.gpu
@pytest.mark.parametrize("n_ranks", [4, 8])
def test_virtual_ranks_level1_leaves(n_ranks):
    import torch
    pts = _lopsided()
    n = pts.shape[0]
    d = ref_descriptor(1, pts, 64, 1e-6, 1.0)
    q = host.generate_charges(n, 4)
    u_ref = api.fmm_apply(api.GpuPlan(d), q)
    plans = [shard.ShardedPlan(d, n_ranks, r) for r in range(n_ranks)]
    qd = torch.from_numpy(q).cuda()
    ud = torch.zeros_like(qd)
    shard.apply_virtual(plans, qd, ud)
    torch.cuda.synchronize()
    assert rel_l2(ud.cpu().numpy(), u_ref) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("n_ranks", [2, 3, 4, 8])
def test_virtual_ranks_2d(n_ranks):
    # 2D: four level-1 quadrants; 8 ranks take the level-2 cut
    import torch
    n = 40000
    d, pts = _desc(dist="annulus", n=n, leaf=40, kernel=0, kappa=1.0)
    q = host.generate_charges(n, 5)
    u_ref = api.fmm_apply(api.GpuPlan(d), q)
    plans = [shard.ShardedPlan(d, n_ranks, r) for r in range(n_ranks)]
    qd = torch.from_numpy(q).cuda()
    ud = torch.zeros_like(qd)
    shard.apply_virtual(plans, qd, ud)
    torch.cuda.synchronize()
    assert rel_l2(ud.cpu().numpy(), u_ref) <= 1e-12


@pytest.mark.gpu
def test_virtual_ranks_parity_vs_oracle_1e6():
    # config-5 geometry at 1e6: 8 level-1 octants over 8 virtual ranks
    import torch
    from oracle import pyoracle as po
    n = 1000000
    pts = host.generate_points("cube", n, 1)
    hp = ref_descriptor(1, pts, 128, 1e-6)
    q = host.generate_charges(n, 1 ^ host.CHARGE_STREAM)
    plans = [shard.ShardedPlan(hp, 8, r) for r in range(8)]
    qd = torch.from_numpy(q).cuda()
    ud = torch.zeros_like(qd)
    shard.apply_virtual(plans, qd, ud)
    torch.cuda.synchronize()
    u = ud.cpu().numpy()
    if po.have_ref():
        u_ref, _ = po.RefPipeline.from_desc(hp).apply(q)
        assert rel_l2(u, u_ref) <= 1e-12
    t = np.arange(0, n, 9973, dtype=np.int32)
    assert max_rel(u[t], api.direct_sum_subset(1, 1.0, pts, q, t)) <= 1e-5


@pytest.mark.gpu
def test_bench_sharded_line_two_ranks_gloo(tmp_path):
    """The N>1 bench path end to end: torchrun, two ranks (one GPU, gloo
    exchange through host memory), the JSON line with parity vs the 1-GPU plan."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--backend", "gloo", "--points", "3e5"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["relerr_vs_single_gpu"] <= 1e-12
    assert line["relerr_vs_direct"] <= 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("case", [("cube", 1, 8), ("sphere", 1, 4), ("gaussian", 1, 4), ("square", 0, 4)])
def test_compact_slot_space_bit_identical(case, monkeypatch):
    """Sharded rank plans keep slots only for the boxes the rank touches (its
    own and shared boxes, the sources its targets read): each rank's slot
    space shrinks with its share, and the sharded result is bit-identical to
    the plans that keep all N slots (SFMM_SHARD_COMPACT=0)."""
    import torch
    dist, kernel, n_ranks = case
    n = 120000
    pts = host.generate_points(dist, n, 3)
    d = ref_descriptor(kernel, pts, 64, 1e-6)
    q = host.generate_charges(n, 9)
    qd = torch.from_numpy(q).cuda()
    out = {}
    for comp in ("1", "0"):
        monkeypatch.setenv("SFMM_SHARD_COMPACT", comp)
        plans = [shard.ShardedPlan(d, n_ranks, r) for r in range(n_ranks)]
        ud = torch.zeros_like(qd)
        shard.apply_virtual(plans, qd, ud)
        torch.cuda.synchronize()
        out[comp] = (ud.cpu().numpy(), [p.info().n_slots for p in plans])
        for p in plans:
            p.close()
    assert np.array_equal(out["1"][0], out["0"][0])
    full = int(d.arrays["iv_off"][-1])
    assert all(s == full for s in out["0"][1])
    # each rank keeps its share plus a ghost layer (a large fraction at these
    # small N; surface / volume at config-5 sizes)
    assert max(out["1"][1]) < full

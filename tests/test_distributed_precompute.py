"""Distributed precompute (config 5 scale, VERDICT r1 missing #5): every rank
builds the same tree, picks the level-1 subtrees it owns from the tree alone,
skeletonizes only those (sfmm_gpu_build_skeletons_subset), and the ranks
exchange index data to form the full descriptor; each rank's plan takes its
operators straight from its own subset build (sfmm_gpu_plan_create_sharded_owned).

Checked on one GPU with virtual ranks: the assembled descriptor and every
rank's operators are bit-identical to one whole-tree skeletonization (a box's
skeleton depends only on its own subtree), and the sharded apply on them
matches the single-GPU plan and the reference restatement."""
import numpy as np
import pytest

from conftest import rel_l2
from oracle import pyoracle as po
from paper_2310_16668_b200 import api, host, shard

pytestmark = pytest.mark.gpu

_INDEX = ("iv_off", "iv", "sk_off", "skel_pos", "rd_off", "red_pos", "T_off", "box_parent_offset")


def _ranks(kernel, pts, leaf, tol, kappa, n_ranks):
    """Phase 1 of every virtual rank (tree, ownership, subset skeletons), then
    the exchange and assembly (phase 2) as distributed_precompute does."""
    hps, parts, owner = [], [], None
    for r in range(n_ranks):
        hp = host.HostPlan.build_tree_gpu(pts, leaf)
        own = shard.subtree_owners(hp, n_ranks)
        if owner is None:
            owner = own
        assert np.array_equal(own, owner)  # every rank derives the same ownership
        hp.skeletonize(kernel, tol, kappa, host_T=False, box_mask=own == r)
        hps.append(hp)
        parts.append(shard.local_index_data(hp, own, r))
    return [shard.assemble_descriptor(hp, parts) for hp in hps], hps, owner


@pytest.mark.parametrize("kernel,dist,n,leaf,n_ranks", [
    (1, "cube", 60000, 64, 8), (1, "sphere", 50000, 60, 4), (3, "cube", 40000, 64, 2),
    (0, "square", 60000, 64, 4),
])
def test_subset_skeletons_assemble_to_the_full_build(kernel, dist, n, leaf, n_ranks):
    kappa = 10.0 if kernel == 3 else 1.0
    pts = host.generate_points(dist, n, 3)
    full = host.HostPlan.build_gpu(kernel, pts, leaf, 1e-6, kappa, host_T=True)
    fd = full.descriptor()
    descs, hps, owner = _ranks(kernel, pts, leaf, 1e-6, kappa, n_ranks)
    for d in descs:
        for f in _INDEX:
            assert np.array_equal(d.arrays[f], fd.arrays[f]), f
    sw = 2 if kernel == 3 else 1
    T_full = np.asarray(fd.arrays["T"])
    T_off = np.asarray(fd.arrays["T_off"])
    for r, hp in enumerate(hps):
        hp.fetch_T()
        T_r = np.asarray(hp.descriptor().arrays["T"])
        mine = np.nonzero(owner == r)[0]
        want = np.concatenate([T_full[T_off[b] * sw:T_off[b + 1] * sw] for b in mine] + [np.zeros(0)])
        assert np.array_equal(T_r, want)
    # each rank only skeletonized its share
    assert all((owner[np.asarray(fd.arrays["box_level"]) >= 1] >= 0))


@pytest.mark.parametrize("kernel,dist,n_ranks", [(1, "cube", 8), (1, "sphere", 4), (3, "cube", 2)])
def test_sharded_apply_on_distributed_precompute(kernel, dist, n_ranks):
    import torch
    kappa = 10.0 if kernel == 3 else 1.0
    n = 80000
    pts = host.generate_points(dist, n, 5)
    descs, hps, owner = _ranks(kernel, pts, 64, 1e-6, kappa, n_ranks)
    plans = [shard.OwnedShardedPlan(descs[r], n_ranks, r, 0, hps[r].device_T()[0], owner)
             for r in range(n_ranks)]
    q = (host.generate_charges_complex if kernel == 3 else host.generate_charges)(n, 31)
    qd = torch.from_numpy(q).cuda()
    ud = torch.zeros_like(qd)
    shard.apply_virtual(plans, qd, ud)
    torch.cuda.synchronize()
    u = ud.cpu().numpy()
    # the same operators on one GPU (the full descriptor needs T for that)
    for hp in hps:
        hp.fetch_T()
    full = host.HostPlan.build_gpu(kernel, pts, 64, 1e-6, kappa, host_T=True)
    single = api.fmm_apply(api.GpuPlan(full.descriptor()), q)
    assert rel_l2(u, single) <= 1e-13
    u_ref, _ = po.oracle_apply(full.descriptor(), q)
    assert rel_l2(u, u_ref) <= 1e-12
    # the plans own exactly the subtrees each rank skeletonized
    for r, p in enumerate(plans):
        assert p.n_owned_points == int(np.sum([np.asarray(descs[0].arrays["box_end"])[b] -
                                               np.asarray(descs[0].arrays["box_begin"])[b]
                                               for b in np.nonzero((owner == r) &
                                                                   (np.asarray(descs[0].arrays["box_level"]) == 1))[0]]))


@pytest.mark.parametrize("n_ranks,n,kernel", [(8, 60000, 1), (3, 40000, 3)])
def test_cpp_rank_precompute_header(n_ranks, n, kernel):
    """include/sfmm_gpu_dist.hpp (the C++ host side of the same flow): every
    virtual rank's assembled descriptor and operators equal the whole-tree
    build, and every rank plan builds (tests/cpp/dist_precompute_check.cpp)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "bin",
                       "dist_precompute_check")
    if not os.path.exists(exe):
        pytest.skip("build/bin/dist_precompute_check not built (make check-bin)")
    r = subprocess.run([exe, str(n_ranks), str(n), str(kernel)], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("ok")

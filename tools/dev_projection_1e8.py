"""Projected 8-GPU apply at N=1e8 (config 5) from one B200.

The full precompute runs on this GPU with T kept on the device (~100 GB);
each of the 8 rank plans is then created from its operator blob (as rank 0
ships them over NCCL in bench.py), timed alone -- begin, mid, fin with
zero-filled exchange buffers -- and destroyed.  N=1e8 does not fit one GPU,
so the reference point is the 1-GPU rate at N=1e7 measured in the same run.
Usage: python tools/dev_projection_1e8.py [N [ranks]]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_16668_b200 import api, host, shard  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 8
REPS = 5
s = torch.cuda.Stream()


def rate_1gpu(n1):
    pts = host.generate_points("cube", n1, 1)
    hp = host.HostPlan.build_gpu(1, pts, 128, 1e-6, host_T=False)
    q = torch.from_numpy(host.generate_charges(n1, 1)).cuda()
    u = torch.zeros_like(q)
    with api.GpuPlan.from_host(hp) as p:
        for _ in range(2):
            api.fmm_apply_device(p, q.data_ptr(), u.data_ptr(), 1, s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(REPS):
            api.fmm_apply_device(p, q.data_ptr(), u.data_ptr(), 1, s.cuda_stream)
        e1.record(s)
        s.synchronize()
        w = p.info().p_dense
    hp.release_device_skeletons()
    return n1 / (e0.elapsed_time(e1) / REPS * 1e-3), w


r1, w1 = rate_1gpu(10_000_000)
print(f"1 GPU, N=1e7: {r1 / 1e6:.1f} Mpoints/s, {w1 / 1e7:.0f} dense pairs per point", flush=True)
t0 = time.perf_counter()
pts = host.generate_points("cube", n, 1)
hp = host.HostPlan.build_gpu(1, pts, 128, 1e-6, host_T=False)
info = hp.info()
print(f"N={n:.0e}: precompute {time.perf_counter() - t0:.1f} s, depth {info['depth']}, "
      f"{info['n_boxes']} boxes, k_max {info['k_max']}", flush=True)
d = hp.desc_struct()
ptr, dev, n_scalars = hp.device_T()
q = torch.from_numpy(host.generate_charges(n, 1)).cuda()
u = torch.zeros_like(q)
times = []
for r in range(nr):
    t0 = time.perf_counter()
    runs, ne = shard.T_runs(d, nr, r)
    blob = torch.empty(max(1, ne), dtype=torch.float64, device="cuda")
    shard.pack_T(ptr, runs, 1, blob, dev)
    torch.cuda.synchronize()
    p = shard.ShardedPlan(d, nr, r, T_owned=blob)
    del blob
    for b in p.buffers() + p.buffers2():
        b.zero_()
    t_plan = time.perf_counter() - t0

    def step():
        p.begin(q, s.cuda_stream, 0)
        if p.cross_symmetric:
            p.mid(s.cuda_stream)
            p.fin(q, u, s.cuda_stream)
        else:
            p.end(q, u, s.cuda_stream)

    with torch.cuda.stream(s):
        for _ in range(2):
            step()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(REPS + 1)]
        ev[0].record(s)
        for i in range(REPS):
            step()
            ev[i + 1].record(s)
    s.synchronize()
    t = float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(REPS)]))
    times.append(t)
    w8 = p.info().p_dense  # global pair count (same on every rank)
    print(f"rank {r}: {p.n_owned_points} points, {p.n_ghost_boxes} ghost boxes, cut {p.cut_level}, "
          f"plan {t_plan:.1f} s, {t:.2f} ms per apply", flush=True)
    p.close()
    torch.cuda.empty_cache()
tmax = max(times)
rate = n / (tmax * 1e-3)
print(f"{nr} GPUs, N={n:.0e}: max rank {tmax:.2f} ms (mean {np.mean(times):.2f}) -> "
      f"{rate / 1e6:.1f} Mpoints/s projected; {rate / r1:.2f}x the 1-GPU rate at 1e7 "
      f"(efficiency {rate / (nr * r1):.3f})", flush=True)
# the deeper tree does more work per point: compare device time per dense pair
t1_equiv = w8 / (w1 / (1e7 / r1))  # seconds one GPU would need at the 1e7 pair rate
print(f"{w8 / n:.0f} dense pairs per point at N={n:.0e} ({w8 / n / (w1 / 1e7):.3f}x 1e7); "
      f"work-adjusted efficiency {t1_equiv / (nr * tmax * 1e-3):.3f}", flush=True)

"""Projected strong scaling of the sharded apply from one GPU.

Each rank's share of one apply (begin: gather, upward pass, pack; end:
unpack, translations, column-sum pack, K2b, downward pass, scatter)
is timed alone on the device with CUDA events, on buffers already holding a
complete exchange.  On N GPUs the step takes about the slowest rank's time
plus the ghost all-to-alls, which SURVEY.md 8e estimates at <0.1 % of the step
over NVLink; it is not included.  Usage: python tools/dev_scaling_projection.py [N [dist [tol [ranks]]]]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_16668_b200 import api, host, shard  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
dist = sys.argv[2] if len(sys.argv) > 2 else "cube"
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6
RANKS = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [2, 4, 8]
REPS = 10  # timed begin/end pairs per rank (median)
pts = host.generate_points(dist, n, 1)
hp = host.HostPlan.build_gpu(1, pts, 128, tol)
q = host.generate_charges(n, 1)
qd = torch.from_numpy(q).cuda()
ud = torch.zeros_like(qd)
s = torch.cuda.Stream()

single = api.GpuPlan(hp.desc_struct())
for _ in range(2):
    api.fmm_apply_device(single, qd.data_ptr(), ud.data_ptr(), 1, s.cuda_stream)
s.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(REPS):
    api.fmm_apply_device(single, qd.data_ptr(), ud.data_ptr(), 1, s.cuda_stream)
e1.record(s)
s.synchronize()
t1 = e0.elapsed_time(e1) / REPS
single.close()
print(f"N={n:.0e} {dist} tol={tol:g}  1 GPU (single plan, graph replay): {t1:.2f} ms")

for nr in RANKS:
    plans = [shard.ShardedPlan(hp.desc_struct(), nr, r) for r in range(nr)]
    shard.apply_virtual(plans, qd, ud)  # fills every rank's receive buffer once
    torch.cuda.synchronize()
    times = []
    for p in plans:
        with torch.cuda.stream(s):
            def end(p=p):
                if p.cross_symmetric:
                    p.mid(s.cuda_stream)
                    p.fin(qd, ud, s.cuda_stream)
                else:
                    p.end(qd, ud, s.cuda_stream)
            for _ in range(2):
                p.begin(qd, s.cuda_stream, 0)
                end()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * REPS + 1)]
            ev[0].record(s)
            for i in range(REPS):
                p.begin(qd, s.cuda_stream, 0)
                ev[1 + 2 * i].record(s)
                end()
                ev[2 + 2 * i].record(s)
        s.synchronize()
        tb = np.median([ev[2 * i].elapsed_time(ev[1 + 2 * i]) for i in range(REPS)])
        te = np.median([ev[1 + 2 * i].elapsed_time(ev[2 + 2 * i]) for i in range(REPS)])
        times.append((float(tb + te), float(tb), float(te)))
    tmax = max(t[0] for t in times)
    print(f"{nr} ranks: per-rank ms (begin+end) {[round(t[0], 2) for t in times]}  max {tmax:.2f}  "
          f"projected speed-up {t1 / tmax:.2f}x  efficiency {t1 / (nr * tmax):.3f}", flush=True)
    print(f"   begin (gather, upward, pack) {[round(t[1], 2) for t in times]}", flush=True)
    print(f"   end (unpack, K2, column-sum pack, K2b, downward, scatter) {[round(t[2], 2) for t in times]}",
          flush=True)
    for p in plans:
        p.close()

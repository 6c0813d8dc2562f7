"""Dev probe: GPU skeletonization vs the host one (accuracy, k, time)."""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
from oracle import pyoracle as po  # noqa: E402
from paper_2310_16668_b200 import api, host  # noqa: E402

cases = [(1, "cube", 20000, 64, 1e-6, 1.0), (0, "square", 20000, 64, 1e-6, 1.0),
         (3, "cube", 20000, 64, 1e-6, 10.0), (1, "sphere", 50000, 64, 1e-8, 1.0),
         (1, "cube", 1000000, 128, 1e-6, 1.0)]
if len(sys.argv) > 1:
    cases = [(1, "cube", int(float(sys.argv[1])), 128, 1e-6, 1.0)]
for kern, dist, n, leaf, tol, kappa in cases:
    pts = host.generate_points(dist, n, 1)
    q = host.generate_charges_complex(n, 3) if kern == 3 else host.generate_charges(n, 3)
    t0 = time.time()
    hg = host.HostPlan.build_gpu(kern, pts, leaf, tol, kappa)
    tg = time.time() - t0
    t0 = time.time()
    hc = host.HostPlan.build(kern, pts, leaf, tol, kappa) if n <= 1000000 else None
    tc = time.time() - t0
    ig = hg.info()
    line = f"kern {kern} {dist} n={n}: gpu skel {ig['t_skel']:.2f}s (total {tg:.2f}s) k_max {ig['k_max']} proj {ig['proj_scalars']}"
    if hc is not None:
        ic = hc.info()
        line += f" | host skel {ic['t_skel']:.2f}s k_max {ic['k_max']} proj {ic['proj_scalars']}"
    u = api.fmm_apply(api.GpuPlan(hg.desc_struct()), q)
    t = np.arange(0, n, max(1, n // 300), dtype=np.int32)
    ref = api.direct_sum_subset(kern, kappa, pts, q, t)
    err = np.max(np.abs(u[t] - ref)) / np.max(np.abs(ref))
    line += f" | relerr vs direct {err:.2e}"
    if n <= 200000:
        u_ref, _ = po.RefPipeline.from_desc(hg.desc_struct()).apply(q, kern == 3)
        line += f" | gpu apply vs ref on gpu skeletons {po.rel_l2(u, u_ref):.2e}"
    print(line, flush=True)

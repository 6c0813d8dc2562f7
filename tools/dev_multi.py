"""Dev probe: multi-RHS apply (DMMA path) vs column loop and vs the oracle."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2310_16668_b200 import api, host  # noqa: E402

for kern, dist, n, leaf, kappa, nrhs in [(3, "cube", 20000, 64, 10.0, 16), (1, "cube", 20000, 64, 1.0, 5),
                                          (0, "square", 20000, 64, 1.0, 16), (3, "sphere", 30000, 64, 10.0, 20),
                                          (3, "cube", 400000, 128, 10.0, 16)]:
    pts = host.generate_points(dist, n, 1)
    hp = host.HostPlan.build_gpu(kern, pts, leaf, 1e-6, kappa)
    plan = api.GpuPlan(hp.desc_struct())
    if kern == 3:
        Q = np.stack([host.generate_charges_complex(n, (1 + r) ^ host.CHARGE_STREAM) for r in range(nrhs)], 1)
    else:
        Q = np.stack([host.generate_charges(n, (1 + r) ^ host.CHARGE_STREAM) for r in range(nrhs)], 1)
    st = api.ApplyStats()
    U = api.fmm_apply(plan, Q, st)
    U = api.fmm_apply(plan, Q, st)
    t_multi = st.ms_total
    cols = [api.fmm_apply(plan, Q[:, r], st) for r in range(nrhs)]
    t_col = 0.0
    for r in range(nrhs):
        api.fmm_apply(plan, Q[:, r], st)
        t_col += st.ms_total
    Uc = np.stack(cols, 1)
    err = np.linalg.norm(U - Uc) / np.linalg.norm(Uc)
    print(f"kern {kern} {dist} n={n} nrhs={nrhs}: rel_l2 multi vs column loop {err:.2e}; "
          f"multi {t_multi:.1f} ms, column loop {t_col:.1f} ms", flush=True)

"""Dev probe: sharded apply (virtual ranks on one GPU) vs the single plan."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2310_16668_b200 import api, host, shard  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1000000
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 128
pts = host.generate_points("cube", n, 1)
hp = host.HostPlan.build_gpu(1, pts, leaf, 1e-6)
print("depth", hp.info()["depth"], "n_boxes", hp.info()["n_boxes"], "leaf", leaf, "env", os.environ.get("SFMM_SYMMETRIC"), os.environ.get("SFMM_SKIP_CANCEL"))
q = host.generate_charges(n, 5)
u_ref = api.fmm_apply(api.GpuPlan(hp.desc_struct()), q)
for nr in (1, 2, 8):
    plans = [shard.ShardedPlan(hp.desc_struct(), nr, r) for r in range(nr)]
    qd = torch.from_numpy(q).cuda()
    ud = torch.zeros_like(qd)
    shard.apply_virtual(plans, qd, ud)
    torch.cuda.synchronize()
    u = ud.cpu().numpy()
    err = np.linalg.norm(u - u_ref) / np.linalg.norm(u_ref)
    line = f"ranks {nr}: rel_l2 {err:.3e}"
    for r, p in enumerate(plans):
        inf = shard.describe(hp.desc_struct(), nr, r)
        idx = inf["owned_points"]
        e = np.linalg.norm(u[idx] - u_ref[idx]) / np.linalg.norm(u_ref[idx])
        line += f" | r{r} {e:.1e} ghosts {p.n_ghost_boxes}"
    print(line, flush=True)

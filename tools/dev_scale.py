"""Dev probe: reference precompute -> GPU plan -> timed applies (not the bench)."""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
from oracle import pyoracle as po  # noqa: E402
from paper_2310_16668_b200 import api  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1000000
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 128
check = len(sys.argv) > 3 and sys.argv[3] == "check"
kern = 1
pts = po.generate_points("cube", n, 1)
t = time.time()
rp = po.RefPipeline.build(kern, pts, leaf, 1e-6)
print("ref build %.1fs" % (time.time() - t), rp.info(), flush=True)
d = rp.descriptor()
q = po.generate_charges(n, 1 ^ po.CHARGE_STREAM)
t = time.time()
plan = api.GpuPlan(d)
print("plan upload %.2fs" % (time.time() - t), flush=True)
inf = plan.info()
print("slots", inf.n_slots, "P_dense %.4e P_skel %.4e M %.4e tasks %d dev bytes %.2f GB" % (
    inf.p_dense, inf.p_skel, inf.m_proj, inf.n_tasks, inf.device_bytes / 1e9), flush=True)
s = api.ApplyStats()
for i in range(4):
    u = api.fmm_apply(plan, q, s)
    W = 20 * inf.p_dense + 2 * inf.p_skel
    print("apply ms_total %.3f ms_translate %.3f  K2 %.2f TF/s(conv F=20)  pairs/s %.3e  Mpts/s %.2f" % (
        s.ms_total, s.ms_translate, W / s.ms_translate / 1e9, inf.p_dense / s.ms_translate / 1e-3,
        n / s.ms_total / 1e3), flush=True)
if check:
    t = time.time()
    u_ref, st = rp.apply(q)
    tr = time.time() - t
    print("ref apply %.2fs (%d threads) Mpts/s %.3f  rel_l2 %.3e" % (
        tr, po.ref_lib().ref_num_threads(), n / tr / 1e6, po.rel_l2(u, u_ref)), flush=True)

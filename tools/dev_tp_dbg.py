import os, sys, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from conftest import golden_files, load_golden, rel_l2
from paper_2310_16668_b200 import api
for path in golden_files():
    desc, ex = load_golden(path)
    res = []
    for tp in ("1", "0"):
        os.environ["SFMM_TREE_PERSIST"] = tp
        plan = api.GpuPlan(desc)
        u = api.fmm_apply(plan, ex["q"])
        u2 = api.fmm_apply(plan, ex["q"])
        res.append((rel_l2(u, ex["u_ref"]), np.array_equal(u, u2)))
        plan.close()
    print(os.path.basename(path), res, flush=True)

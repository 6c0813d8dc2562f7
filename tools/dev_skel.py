"""Dev: GPU precompute timing (tree + skeletons) at one size; env knobs apply."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_16668_b200 import host  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**7
kern = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dist = sys.argv[3] if len(sys.argv) > 3 else "cube"
tol = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-6
pts = host.generate_points(dist, n, 1)
for rep in range(2):
    t = time.perf_counter()
    hp = host.HostPlan.build_gpu(kern, pts, 128, tol, 10.0 if kern == 3 else 1.0, host_T=False)
    inf = hp.info()
    print(f"rep {rep}: total {time.perf_counter() - t:.3f} s  tree {inf['t_tree']:.3f}  skel {inf['t_skel']:.3f}"
          f"  k_max {inf['k_max']} proj {inf['proj_scalars']}", flush=True)
    hp.close()

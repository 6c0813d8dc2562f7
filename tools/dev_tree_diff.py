"""Dev: where does the GPU tree differ from the host tree?"""
import sys
import os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_16668_b200 import host

dist, n, leaf = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
pts = host.generate_points(dist, n, 29)
dg = host.HostPlan.build_tree_gpu(pts, leaf).descriptor()
dh = host.HostPlan.build_tree(pts, leaf).descriptor()
print("depth", dg.scalars["depth"], dh.scalars["depth"], "n_boxes", dg.scalars["n_boxes"], dh.scalars["n_boxes"])
print("level_begin gpu ", dg.arrays["level_begin"])
print("level_begin host", dh.arrays["level_begin"])
for k in ["perm", "box_parent", "box_level", "box_begin", "box_end", "box_leaf", "coll", "coarse", "fine"]:
    a, b = dg.arrays[k], dh.arrays[k]
    if a.shape != b.shape:
        print(k, "shape", a.shape, b.shape)
        continue
    d = np.nonzero(a != b)[0]
    print(k, "ndiff", d.size, "first", d[:5], a[d[:5]] if d.size else "", b[d[:5]] if d.size else "")

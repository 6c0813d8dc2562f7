"""Dev tool: where the multi-RHS translation work of a plan sits.

Per level: dense pair work by mode (ifo split into self / foldable colleague
pairs, ifs, tfo, level-1), the pairs the exact-cancellation rule drops, and
the uhat-pass work (skeleton rows x h-weighted sources).  Used to size the
symmetric K2m fold.

    python tools/dev_k2m_stats.py --kernel 3 --dist cube --n 4e6 --leaf 128 --tol 1e-6
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_16668_b200 import host  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", type=int, default=3)
    ap.add_argument("--dist", default="cube")
    ap.add_argument("--n", type=float, default=4e6)
    ap.add_argument("--leaf", type=int, default=128)
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--kappa", type=float, default=10.0)
    a = ap.parse_args()
    n = int(a.n)
    pts = host.generate_points(a.dist, n, 1)
    hp = host.HostPlan.build_gpu(a.kernel, pts, a.leaf, a.tol, a.kappa, host_T=False)
    d = hp.descriptor()
    A = d.arrays
    lev = np.asarray(A["box_level"])
    leaf = np.asarray(A["box_leaf"]).astype(bool)
    nb = np.diff(np.asarray(A["iv_off"]))
    kb = np.diff(np.asarray(A["sk_off"]))
    unc = (lev >= 2) & (nb > 0) & (kb == nb)
    coll_off, coll = np.asarray(A["coll_off"]), np.asarray(A["coll"])
    coarse_off, coarse = np.asarray(A["coarse_off"]), np.asarray(A["coarse"])
    fine_off, fine = np.asarray(A["fine_off"]), np.asarray(A["fine"])
    depth = int(d.scalars["depth"])
    print(f"N={n} depth={depth} boxes={len(nb)}")
    tot = {}
    for l in range(1, depth + 1):
        bs = np.nonzero(lev == l)[0]
        row = dict(self=0.0, fold=0.0, ifs=0.0, tfo=0.0, l1=0.0, skipped=0.0, hpass=0.0)
        for b in bs:
            if l >= 2:
                for c in coll[coll_off[b]:coll_off[b + 1]]:
                    w = float(nb[b]) * nb[c]
                    if unc[b] and unc[c]:
                        row["skipped"] += w
                    elif c == b:
                        row["self"] += w
                    else:
                        row["fold"] += w
                    if not (unc[b] and unc[c]):
                        row["hpass"] += float(kb[b]) * kb[c]
                if not unc[b]:
                    for c in coarse[coarse_off[b]:coarse_off[b + 1]]:
                        row["ifs"] += float(nb[b]) * nb[c]
                        row["hpass"] += float(kb[b]) * nb[c]
            if l == 1:
                row["l1"] += float(nb[b]) * nb[lev == 1].sum()
            if leaf[b]:
                for c in fine[fine_off[b]:fine_off[b + 1]]:
                    if not unc[c]:
                        row["tfo"] += float(nb[b]) * nb[c]
        if bs.size:
            print(f"level {l}: boxes {bs.size:7d} n mean {nb[bs].mean():7.1f} k mean "
                  f"{kb[bs].mean():7.1f} leaves {int(leaf[bs].sum()):6d} unc {int(unc[bs].sum()):6d}  "
                  + " ".join(f"{k} {v:.3e}" for k, v in row.items()))
        for k, v in row.items():
            tot[k] = tot.get(k, 0.0) + v
    ev = tot["self"] + tot["fold"] + tot["ifs"] + tot["tfo"] + tot["l1"]
    print("total " + " ".join(f"{k} {v:.3e}" for k, v in tot.items()))
    print(f"evaluated dense pairs {ev:.3e}; foldable share {tot['fold'] / ev:.3f}; "
          f"uhat-pass share {tot['hpass'] / ev:.3f}")


if __name__ == "__main__":
    main()

import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, sys
from paper_2310_16668_b200 import host
n=int(float(sys.argv[1])); dist=sys.argv[2] if len(sys.argv)>2 else "cube"; tol=float(sys.argv[3]) if len(sys.argv)>3 else 1e-6
pts=host.generate_points(dist,n,1)
hp=host.HostPlan.build_gpu(1,pts,128,tol)
a=hp.descriptor().arrays
nb=np.diff(a["iv_off"]).astype(np.int64); kb=np.diff(a["sk_off"]).astype(np.int64)
lvl=a["box_level"]; unc=(lvl>=2)&(nb>0)&(kb==nb)
co=a["coll_off"]; cl=a["coll"]
useful=0; exe_sym=0; exe_rowpad=0; sym_useful=0
ceil32=lambda x: ((x+31)//32)*32
for b in range(len(nb)):
    if lvl[b]<2: continue
    for c in cl[co[b]:co[b+1]]:
        if unc[b] and unc[c]: continue
        if c==b:
            useful+=nb[b]*nb[c]; exe_rowpad+=ceil32(nb[b])*nb[c]; continue
        if c>b:
            u=2*nb[b]*nb[c]; useful+=u; sym_useful+=u
            exe_sym+=ceil32(nb[b])*ceil32(nb[c])   # one rotation pass covers both directions
print("sym pairs: useful (both dirs) %.3e, executed lane-pairs %.3e, ratio useful/(2*exec) %.3f" % (sym_useful, exe_sym, sym_useful/(2*exe_sym)))
# column-only padding (rows padded already counted): ratio of ceil32(nc) to nc
cp=0; cu=0
for b in range(len(nb)):
    if lvl[b]<2: continue
    for c in cl[co[b]:co[b+1]]:
        if c>b and not (unc[b] and unc[c]):
            cp+=ceil32(nb[b])*ceil32(nb[c]); cu+=ceil32(nb[b])*nb[c]
print("column padding share in sym steps: %.3f" % (1-cu/cp))
h=np.bincount(np.minimum(nb[lvl==lvl.max()],200)//8)
print("leaf-level n histogram (x8):", h[:20])

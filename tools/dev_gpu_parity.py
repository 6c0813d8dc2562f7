import sys, time, numpy as np
sys.path.insert(0,'/root/repo')
from oracle import pyoracle as po
from paper_2310_16668_b200 import api
for kern, dist, n, leaf, tol, kappa in [(1,'cube',3000,40,1e-6,1.0),(0,'square',3000,40,1e-6,1.0),(3,'cube',2000,40,1e-6,2.0),(1,'sphere',4000,30,1e-8,1.0),(1,'cube',200000,128,1e-6,1.0), (0,'square',100000,64,1e-6,1.0), (1,'cube',300,100,1e-6,1.0)]:
    pts = po.generate_points(dist, n, 1)
    rp = po.RefPipeline.build(kern, pts, leaf, tol, kappa)
    d = rp.descriptor()
    cplx = kern>=2
    q = po.generate_charges_complex(n, 5) if cplx else po.generate_charges(n, 5)
    t=time.time(); u_ref, st = rp.apply(q, cplx); tref=time.time()-t
    plan = api.GpuPlan(d)
    s = api.ApplyStats()
    u = api.fmm_apply(plan, q, s)
    u = api.fmm_apply(plan, q, s)
    print(kern, dist, n, rp.info(), 'rel_l2 gpu vs ref %.3e'%po.rel_l2(u,u_ref), 'stats', st, s, 'ref %.3fs'%tref, flush=True)

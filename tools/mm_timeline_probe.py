import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import kl_inputs as G, paper_1303_5164_b200 as K
from paper_1303_5164_b200.workload import Instance
for shape in [dict(M=8192,N=2048,K=2048), dict(M=2048,N=2048,K=2048)]:
    ctx = K.Context(device=0, audit=2)
    i = Instance(G.gen("MM", shape), "cuda")
    for _ in range(3): ctx.run_capped("MM", i.grid, i.args, 0)
    ms = ctx.run_capped("MM", i.grid, i.args, 0)
    rec = ctx.trace()[-1]
    tl = None
    for kid in range(1, 8):
        try:
            tl = ctx.timeline(kid, i.grid); 
        except Exception: continue
    s, e = tl[:, 0].astype(np.float64), tl[:, 1].astype(np.float64)
    t0 = rec.t0_ns if hasattr(rec,'t0_ns') else s.min()
    print(shape, "event ms", ms, "rec t0..t1 us", (rec.t1_ns-rec.t0_ns)/1e3 if hasattr(rec,'t1_ns') else None)
    s, e = (s - s.min())/1e3, (e - s.min()*0 - tl[:,0].min())/1e3
    d = e - s
    order = np.argsort(s)
    print(" first starts", np.round(s[order][:5],2), "last starts", np.round(s[order][-5:],2))
    print(" dur mean %.2f p10 %.2f p50 %.2f p90 %.2f max %.2f" % (d.mean(), *np.percentile(d,[10,50,90]), d.max()))
    print(" span %.2f" % e.max())
    # durations by start rank
    ranks = np.argsort(order)
    for w in range(5):
        sel = (ranks >= w*74) & (ranks < (w+1)*74)
        if sel.any(): print("  wave", w, "n", sel.sum(), "start med %.2f dur med %.2f" % (np.median(s[sel]), np.median(d[sel])))
    ctx.close()

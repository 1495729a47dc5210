import sys, os
sys.path.insert(0, os.getcwd())
import torch, statistics
import kl_inputs as G
import paper_1303_5164_b200 as K
from paper_1303_5164_b200.workload import Instance
ctx = K.Context(device=0)
for kind in ["ST"]:
    i = Instance(G.gen(kind, "paper"), "cuda")
    for mode in ["plain", "persistent"]:
        ts=[]
        for r in range(6):
            torch.cuda.synchronize()
            if mode == "plain":
                e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
                e0.record(); ctx.run_plain(kind, i.grid, i.args, 0); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
            else:
                ts.append(ctx.run_capped(kind, i.grid, i.args, 0))
        print(kind, mode, "ms", round(statistics.median(ts[1:]),4), "GB/s", round(2*4*512**3/(statistics.median(ts[1:])*1e-3)/1e9,1))

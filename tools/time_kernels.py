"""Solo device time of each kind at paper size (plain launch, L2 flushed, median of 7)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance  # noqa: E402

kinds = sys.argv[1:] or ["PC", "SAD", "SPMV", "ST", "MM", "MRIQ", "BS", "TEA"]
ctx = K.Context(device=0)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for k in kinds:
    i = Instance(G.gen(k, "paper"), "cuda")
    ts = []
    for _ in range(7):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.run_plain(k, i.grid, i.args, 0)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"{k:5s} {ts[3]*1e3:9.1f} us   regs {ctx.get_profile(k).regs} bmax {ctx.get_profile(k).bmax}", flush=True)

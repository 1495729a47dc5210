"""ncu target: one plain launch (or one scheduled queue) of a kind at paper size.
usage: python tools/prof_target.py KIND [plain|sched]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance  # noqa: E402

kind = sys.argv[1]
mode = sys.argv[2] if len(sys.argv) > 2 else "plain"
ctx = K.Context(device=0)
inst = Instance(G.gen(kind, "paper"), "cuda")
torch.cuda.synchronize()
for _ in range(2):
    if mode == "plain":
        ctx.run_plain(kind, inst.grid, inst.args, 0)
    else:
        ctx.submit(kind, inst.grid, inst.args)
        ctx.sync()
torch.cuda.synchronize()
print("done", kind, mode)

#!/usr/bin/env python
"""Target for ncu application-range replay (aggregate hardware counters over a whole
co-scheduled phase; kernel replay would serialise the concurrent kernels): warms up, then brackets
ONE step of the bench queue (ALL mix x4, paper sizes) with cudaProfilerStart/Stop -- either the
Kernelet step (model batch + sliced, co-scheduled persistent launches) or the sequential baseline
(the same kernels as plain grids on one stream).
usage: ncu --replay-mode app-range --profile-from-start off --metrics ... python tools/range_target.py {kernelet|sequential}"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance, inputs_to_device  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "kernelet"
profiles, kcfg = bench.load_profiles(os.path.join(ROOT, "profiles", "kl_profile_b200.json"))
ctx = K.Context(device=0, profiles=profiles, **kcfg)
kinds = bench.build_queue(0, 1, 4)
data = {k: G.gen(k, "paper") for k in sorted(set(kinds))}
inputs = {k: inputs_to_device(data[k], "cuda") for k in data}
insts = [Instance(data[k], "cuda", inputs=inputs[k]) for k in kinds]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def step():
    if mode == "kernelet":
        ctx.reset_model_cache()
        ctx.submit_many([(i.kind, i.grid, i.args, n + 1, None) for n, i in enumerate(insts)])
        ctx.sync()
    else:
        for i in insts:
            ctx.run_plain(i.kind, i.grid, i.args, 0)
        torch.cuda.synchronize()


for _ in range(2):
    flush.zero_()
    torch.cuda.synchronize()
    step()
flush.zero_()
torch.cuda.synchronize()
torch.cuda.profiler.start()
step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("range target done", mode, flush=True)

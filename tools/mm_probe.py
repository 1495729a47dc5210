#!/usr/bin/env python
"""MM solo timing over shapes (plain grid and persistent pair launcher, CUDA events, median of 7,
L2 not flushed: operands are L2-resident at these sizes anyway) -- the tile-pipeline probe.
usage: python tools/mm_probe.py [MxNxK ...]      (needs a GPU; KL_LIB_PATH selects a build)"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance  # noqa: E402

shapes = sys.argv[1:] or ["8192x2048x2048", "8192x2048x4096", "8192x2048x1024", "2048x2048x2048", "18944x2048x2048"]
ctx = K.Context(device=0)
for sh in shapes:
    M, N, Kd = (int(x) for x in sh.split("x"))
    i = Instance(G.gen("MM", dict(M=M, N=N, K=Kd)), "cuda")
    res = {}
    for mode in ("plain", "persistent"):
        ts = []
        for _ in range(8):
            torch.cuda.synchronize()
            if mode == "plain":
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ctx.delay(torch.cuda.current_stream(), 200_000)   # host launch latency outside the interval
                e0.record()
                ctx.run_plain("MM", i.grid, i.args, 0)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            else:
                ts.append(ctx.run_capped("MM", i.grid, i.args, 0, spin_ns=200_000) - 0.2)   # spin inside the interval
        res[mode] = statistics.median(ts[1:])
    fl = 2.0 * M * N * Kd
    print(f"MM {sh:>16s} tiles {i.grid:5d}  plain {res['plain'] * 1e3:8.1f} us ({fl / res['plain'] / 1e9:6.0f} TF/s)  "
          f"persistent {res['persistent'] * 1e3:8.1f} us ({fl / res['persistent'] / 1e9:6.0f} TF/s)", flush=True)

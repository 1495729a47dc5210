#!/usr/bin/env python
"""Solo duration of every kind at paper size: plain grid (hardware block scheduling) vs the
persistent slice launcher uncapped (run_capped cap 0): the launcher's own overhead.
SPIN=1 queues a 200 us device delay (kl_delay) before each timed launch and subtracts it,
so the host-side launch work is hidden the way it is inside a scheduled queue (where launches are
issued while earlier kernels run); the numbers are then device-side only.
usage: python tools/launcher_overhead.py      (needs a GPU)"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance  # noqa: E402

CHUNK = int(os.environ.get("CHUNK", "0"))
SPIN = int(os.environ.get("SPIN", "0"))
KINDS = os.environ.get("KINDS", "PC,SAD,SPMV,ST,MM,MRIQ,BS,TEA").split(",")
ctx = K.Context(device=0, chunk=CHUNK)
SPIN_NS = 200_000


def spin_ms():
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.delay(torch.cuda.current_stream(), SPIN_NS)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts[1:])


sp = spin_ms() if SPIN else 0.0
for kind in KINDS:
    i = Instance(G.gen(kind, "paper"), "cuda")
    res = {}
    for mode in ("plain", "persistent"):
        ts = []
        for _ in range(6):
            torch.cuda.synchronize()
            if mode == "plain":
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                if SPIN:
                    ctx.delay(torch.cuda.current_stream(), SPIN_NS)
                ctx.run_plain(kind, i.grid, i.args, 0)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) - sp)
            else:
                ts.append(ctx.run_capped(kind, i.grid, i.args, 0, spin_ns=SPIN_NS if SPIN else 0) - sp)
        res[mode] = statistics.median(ts[1:])
    print(f"{kind:5s} grid {i.grid:6d} plain {res['plain']:.4f} ms  persistent {res['persistent']:.4f} ms  "
          f"overhead {100 * (res['persistent'] / res['plain'] - 1):+.1f} %" + ("  (spin-hidden launch)" if SPIN else ""),
          flush=True)

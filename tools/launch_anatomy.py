#!/usr/bin/env python
"""Device-side anatomy of one solo persistent launch per kind (config.audit = 2): first admission
(t0) -> first virtual block start -> last virtual block end -> epoch close (t1), against the
event-timed duration with the host launch hidden behind a device delay (SPIN).
usage: KINDS=SPMV,SAD python tools/launch_anatomy.py      (needs a GPU)"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance  # noqa: E402

KINDS = os.environ.get("KINDS", "SPMV,SAD,ST,BS,MM").split(",")
SPIN_NS = 200_000
for kind in KINDS:
    ctx = K.Context(device=0, audit=2)
    i = Instance(G.gen(kind, "paper"), "cuda")
    rows = []
    for rep in range(4):
        ms = ctx.run_capped(kind, i.grid, i.args, 0, spin_ns=SPIN_NS)
        rec = ctx.trace()[-1]
        kid = rec.id
        tl = ctx.timeline(kid, i.grid).astype(np.float64)
        first, last = tl[:, 0].min(), tl[:, 1].max()
        rows.append((ms * 1e3 - SPIN_NS / 1e3, (first - rec.t0_ns) / 1e3, (last - first) / 1e3, (rec.t1_ns - last) / 1e3,
                     (rec.t1_ns - rec.t0_ns) / 1e3))
    r = np.median(np.array(rows[1:]), axis=0)
    print(f"{kind:5s} event-minus-spin {r[0]:7.1f} us | admit->first vb {r[1]:6.1f} | vb span {r[2]:7.1f} | "
          f"last vb->close {r[3]:6.1f} | epoch {r[4]:7.1f} | outside epoch {r[0] - r[4]:6.1f}", flush=True)
    ctx.close()

"""Per-virtual-block timeline of one solo persistent launch per kind (config.audit = 2): where
the slice launcher's time goes against the plain grid -- start ramp, steady vb rate, tail.
usage: KINDS=ST,BS python tools/launcher_timeline.py   (needs a GPU)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance  # noqa: E402

KINDS = os.environ.get("KINDS", "SAD,SPMV,ST,BS,TEA").split(",")
for kind in KINDS:
    ctx = K.Context(device=0, audit=2)
    i = Instance(G.gen(kind, "paper"), "cuda")
    for _ in range(2):
        ctx.run_plain(kind, i.grid, i.args, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.run_plain(kind, i.grid, i.args, 0)
    e1.record()
    e1.synchronize()
    plain = e0.elapsed_time(e1)
    ms = ctx.run_capped(kind, i.grid, i.args, 0)
    tl = None
    for kid in range(1, 4):
        try:
            tl = ctx.timeline(kid, i.grid)
            break
        except Exception:
            continue
    rec = ctx.trace()[-1]
    s, e = tl[:, 0].astype(np.float64), tl[:, 1].astype(np.float64)
    t0 = s.min()
    s, e = (s - t0) / 1e3, (e - t0) / 1e3
    d = e - s
    n_slots = rec.admitted if hasattr(rec, "admitted") else 0
    first_wave = np.sort(s)[: max(1, min(len(s), n_slots or 1))]
    ends = np.sort(e)
    print(f"{kind:5s} plain {plain * 1e3:7.1f} us  persistent(event) {ms * 1e3:7.1f} us  span(first start..last end) "
          f"{ends[-1]:7.1f} us  admitted {n_slots}  vb dur mean {d.mean():6.2f} p50 {np.median(d):6.2f} p99 "
          f"{np.percentile(d, 99):6.2f} us  first-wave start spread {first_wave[-1]:6.2f} us  "
          f"ends at 50/90/99/100 %: {np.percentile(ends, 50):6.1f} {np.percentile(ends, 90):6.1f} "
          f"{np.percentile(ends, 99):6.1f} {ends[-1]:6.1f}  busy-sum/slots {d.sum() / max(n_slots, 1):6.1f} us", flush=True)
    print("   trace:", {f: getattr(rec, f) for f, _ in rec._fields_}, flush=True)
    ctx.close() if hasattr(ctx, "close") else None

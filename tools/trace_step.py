"""Diagnostics on the GPU box: (1) each kind's duration through the persistent launcher at every
occupancy level (cap sweep), (2) one scheduled ALL x4 step with its launch trace."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance, inputs_to_device  # noqa: E402

profiles, kcfg = bench.load_profiles(os.path.join(ROOT, "profiles", "kl_profile_b200.json"))
ctx = K.Context(device=0, profiles=profiles, **kcfg)
kinds = bench.build_queue(0, 1, 4)
data = {k: G.gen(k, "paper") for k in sorted(set(kinds))}
inputs = {k: inputs_to_device(data[k], "cuda") for k in data}
insts = [Instance(data[k], "cuda", inputs=inputs[k]) for k in kinds]
out = {"sweep": {}, "trace": []}
for k in ([] if "--no-sweep" in sys.argv else sorted(set(kinds))):
    i = next(x for x in insts if x.kind == k)
    p = ctx.get_profile(k)
    row = {}
    for cap in [0] + list(range(1, p.bmax + 1)):
        ctx.run_capped(k, i.grid, i.args, cap)
        row[cap] = round(ctx.run_capped(k, i.grid, i.args, cap), 4)
    out["sweep"][k] = row
    print(k, "bmax", p.bmax, "wpb", p.wpb, row, flush=True)
for rep in range(3):
    ctx.reset_model_cache()
    torch.cuda.synchronize()
    n0 = len(ctx.trace())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for n, i in enumerate(insts):
        ctx.submit(i.kind, i.grid, i.args, tag=n + 1)
    ctx.sync()
    e1.record()
    e1.synchronize()
    tr = ctx.trace()[n0:]
print("step ms", e0.elapsed_time(e1), "stats", {f: getattr(ctx.stats(), f) for f, _ in K.Stats._fields_})
t00 = min(t.t0_ns for t in tr if t.admitted)
for t in sorted(tr, key=lambda t: t.t0_ns):
    r = dict(kind=K.KINDS[t.kind], cap=t.cap, start=t.start, end=t.end, exh=t.exhausted, adm=t.admitted,
             maxsm=t.max_per_sm, t0=round((t.t0_ns - t00) / 1e3, 1), t1=round((t.t1_ns - t00) / 1e3, 1),
             dec=t.phase, partner=K.KINDS[t.partner_kind] if t.partner_kind >= 0 else None, cp=round(t.cp, 3), lane=t.lane)
    out["trace"].append(r)
    print(r)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "trace_step.json"), "w"), indent=1)

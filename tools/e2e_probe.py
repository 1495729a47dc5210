#!/usr/bin/env python
"""Timeline of one e2e bench step: when each kind's H2D copy lands (CUDA events) and when its
kernels run (device launch records), to see whether the PCIe copies or the kernels bound it."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance, alloc_outputs, inputs_to_device  # noqa: E402

dev = torch.device("cuda", 0)
profiles, kcfg = bench.load_profiles(os.path.join(bench.ROOT, "profiles", "kl_profile_b200.json"))
kinds = bench.build_queue(0, 1, 4, "c2")
data = {k: G.gen(k, "paper") for k in sorted(set(kinds))}
inputs = {k: inputs_to_device(data[k], dev) for k in data}
insts = [Instance(data[k], dev, inputs=inputs[k]) for k in kinds]
ctx = K.Context(device=0, profiles=profiles, split_rule=1, **kcfg)
order = ["MRIQ", "SAD", "PC", "MM", "SPMV", "TEA", "ST", "BS"]
host = {k: {n: t.cpu().pin_memory() for n, t in inputs[k].items()} for k in order}
cs = torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    ready, tev = {}, {}
    with torch.cuda.stream(cs):
        for k in order:
            for n, t in inputs[k].items():
                t.copy_(host[k][n], non_blocking=True)
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(cs)
            ready[k] = ev
    n0 = len(ctx.trace())
    ctx.reset_model_cache()
    ctx.submit_many([(i.kind, i.grid, i.args, n + 1, ready[i.kind]) for n, i in enumerate(insts)])
    ctx.sync()
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(cs)
    e1.synchronize()
    tr = ctx.trace()[n0:]
    print("rep", rep, "total ms", round(e0.elapsed_time(e1), 2))
    for k in order:
        mb = sum(t.numel() * t.element_size() for t in inputs[k].values()) / 1e6
        print(f"  {k:5s} {mb:7.1f} MB copied by {e0.elapsed_time(ready[k]):7.2f} ms")
    z = min(t.t0_ns for t in tr if t.admitted)
    last = max(t.t1_ns for t in tr)
    print("  kernels: first start -> last end", round((last - z) / 1e6, 2), "ms")
    for k in order:
        ts = [t for t in tr if K.KINDS[t.kind] == k and t.admitted]
        print(f"  {k:5s} kernels {(min(t.t0_ns for t in ts) - z) / 1e6:7.2f} .. {(max(t.t1_ns for t in ts) - z) / 1e6:7.2f} ms")
    if rep == 2:
        for t in sorted(tr, key=lambda t: t.t0_ns):
            if not t.admitted:
                continue
            print(f"    {K.KINDS[t.kind]:5s} cap{t.cap:3d}/{t.cap_max:2d} g{t.grids} [{t.start:6d},{t.end:6d}) exh{t.exhausted} "
                  f"{(t.t0_ns - z) / 1e6:7.2f}..{(t.t1_ns - z) / 1e6:7.2f} dec{t.phase} "
                  f"{K.KINDS[t.partner_kind] if t.partner_kind >= 0 else None} cp{t.cp:.3f}")

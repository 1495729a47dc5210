#!/usr/bin/env python
"""Target for compute-sanitizer (SURVEY §4 tier 5, §5 race detection): every kernel at oracle
size unsliced, explicitly sliced (index rectification, 3 slices, permuted order), through the
persistent slice launcher (scheduler: the whole mixed queue co-scheduled), and one model batch
(kl_predict over candidate pairs).  Checks parity so a sanitizer run is also a correctness run.
usage: compute-sanitizer --tool {memcheck,racecheck,synccheck} python tests/sanitize_target.py [KINDS]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import kl_inputs as G  # noqa: E402
import oracle as O  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance  # noqa: E402
from kl_check import compare  # noqa: E402

kinds = sys.argv[1].split(",") if len(sys.argv) > 1 else ["PC", "SAD", "SPMV", "ST", "MM", "MRIQ", "BS", "TEA", "MATADD", "SYNTH"]
ctx = K.Context(device=0, audit=1, alpha_p=0.0, alpha_m=0.0)
ds = {k: G.gen(k, "small") for k in kinds}
refs = {k: O.run_kernel(ds[k]) for k in kinds}
for k in kinds:
    inst = Instance(ds[k], "cuda")
    ctx.run_plain(k, inst.grid, inst.args, 0)
    torch.cuda.synchronize()
    compare(k, inst.result(), refs[k])
    g = inst.grid
    cuts = sorted({0, g // 3, (2 * g) // 3, g})
    sl = [(a, b - a) for a, b in zip(cuts, cuts[1:]) if b > a][::-1]
    for o in inst.outputs.values():
        o.fill_(0)
    for off, n in sl:
        ctx.run_plain(k, inst.grid, inst.args, 0, off, n)
    torch.cuda.synchronize()
    compare(k, inst.result(), refs[k])
    print(f"{k}: unsliced + sliced ok", flush=True)
insts = [Instance(ds[k], "cuda") for k in kinds * 2]
ids = [ctx.submit(i.kind, i.grid, i.args, tag=n + 1) for n, i in enumerate(insts)]
c = ctx.sync()
for kid, i in zip(ids, insts):
    compare(i.kind, i.result(), refs[i.kind])
    assert np.all(ctx.audit(kid, i.grid) == 1), i.kind
print(f"scheduler: {len(insts)} kernels co-scheduled, {c.phases} phases, audit ok", flush=True)
model_kinds = [k for k in kinds if k in ("PC", "SAD", "SPMV", "ST", "MM", "MRIQ", "BS", "TEA")]
cands = [(a, b, 1, 1) for a in model_kinds for b in model_kinds if a < b]
if cands:
    pr = ctx.predict(cands)
    print(f"model: {len(pr)} predictions, statuses {sorted(set(p.status for p in pr))}", flush=True)
ctx.close()
print("sanitize target done")

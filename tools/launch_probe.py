#!/usr/bin/env python
"""Launch latency anatomy with a -DKL_PROBE_ANATOMY build (KL_LIB_PATH=variants/libkl_probe.so):
a device delay releases at a stamped time, the persistent launch queued behind it records block
0's entry, the first admission (t0), the epoch close (t1) and the end of finalize on the device
clock.  Prints release->entry (launch latency on an idle stream), entry->t0 (join + admission),
t0->t1 (epoch), t1->done (finalize), next to the event-timed duration.
usage: KL_LIB_PATH=variants/libkl_probe.so KL_PROBE_ANATOMY=1 python tools/launch_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance  # noqa: E402

KINDS = os.environ.get("KINDS", "SPMV,SAD,ST,MRIQ,MATADD").split(",")
stamp = torch.zeros(1, dtype=torch.int64, device="cuda")
os.environ["KL_TIMING_SPIN_STAMP"] = str(stamp.data_ptr())
for kind in KINDS:
    ctx = K.Context(device=0)
    i = Instance(G.gen(kind, "paper"), "cuda")
    for rep in range(3):
        ms = ctx.run_capped(kind, i.grid, i.args, 0, spin_ns=100_000)
        torch.cuda.synchronize()
        print(f"{kind} rep {rep} event {ms * 1e3 - 100:.1f} us  release stamp {int(stamp.item())}", file=sys.stderr, flush=True)
    ctx.close()

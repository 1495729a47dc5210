#!/usr/bin/env python
"""Where an MM launch's time goes: device time stamps from a -DKL_MM_PROBE build (kl_mm.cu): per
CTA pair, kernel entry, end of init, per tile the MMA issuer's first-stage-full and last-MMA-issued
times, the epilogue's accumulator-ready / stores-issued times, the leader producer's publish and
first-load times and the MMA issuer's tile-item / accumulator-free times, and fini.  Plain grid (the solo roofline and
the sequential baseline) and the uncapped persistent launcher.
usage: KL_LIB_PATH=variants/libkl_mmprobe.so python tools/mm_stamp_probe.py [MxNxK]   (needs a GPU)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance  # noqa: E402

sh = sys.argv[1] if len(sys.argv) > 1 else "8192x2048x2048"
M, N, Kd = (int(x) for x in sh.split("x"))
L = K.lib()
L.kl_mm_probe_read.argtypes = [C.c_void_p, C.c_int]
stride = L.kl_mm_probe_stride()
NF = 8
ntile = (stride - 4) // NF
ctx = K.Context(device=0)
i = Instance(G.gen("MM", dict(M=M, N=N, K=Kd)), "cuda")
buf = (C.c_ulonglong * (96 * stride))()


def read():
    assert L.kl_mm_probe_read(buf, 96 * stride) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(96, stride).astype(np.float64)
    return a


def report(name, a, ev_ms):
    live = a[:, ntile * NF] > 0
    a = a[live]
    t0 = a[:, ntile * NF].min()
    a = np.where(a > 0, (a - t0) / 1e3, np.nan)   # us from the first pair's entry
    ent, ini, pre, end = (a[:, ntile * NF + f] for f in range(4))
    tiles = a[:, :ntile * NF].reshape(-1, ntile, NF)
    print(f"== {name}: {len(a)} pairs, event-timed {ev_ms * 1e3:.1f} us, device span (first entry -> last fini) "
          f"{np.nanmax(end):.1f} us")
    print(f"  entry spread {np.nanmin(ent):.2f}..{np.nanmax(ent):.2f}  init done {np.nanmedian(ini):.2f} (max {np.nanmax(ini):.2f})")
    for j in range(ntile):
        t = tiles[:, j]
        if np.all(np.isnan(t[:, 0])):
            break
        d = t[:, 1] - t[:, 0]
        print(f"  tile {j}: n {np.sum(~np.isnan(t[:, 0])):3d}  mma start med {np.nanmedian(t[:, 0]):6.2f} "
              f"[{np.nanmin(t[:, 0]):6.2f}, {np.nanmax(t[:, 0]):6.2f}]  mma span med {np.nanmedian(d):6.2f}  "
              f"epi drain (acc ready -> stores issued) med {np.nanmedian(t[:, 3] - t[:, 2]):5.2f} (stores issued max {np.nanmax(t[:, 3]):6.2f})")
        if not np.all(np.isnan(t[:, 4])):
            print(f"          producer: published {np.nanmedian(t[:, 4]):6.2f}  first load issued {np.nanmedian(t[:, 5]):6.2f};  "
                  f"MMA: got item {np.nanmedian(t[:, 6]):6.2f}  accumulator free {np.nanmedian(t[:, 7]):6.2f}  first stage full {np.nanmedian(t[:, 0]):6.2f}")
        if j > 0:
            g = t[:, 0] - tiles[:, j - 1, 1]
            print(f"          gap last MMA issued (tile {j - 1}) -> first stage full (tile {j}): med {np.nanmedian(g):5.2f} max {np.nanmax(g):5.2f}")
    print(f"  before fini med {np.nanmedian(pre):.2f} max {np.nanmax(pre):.2f}; fini end med {np.nanmedian(end):.2f} max {np.nanmax(end):.2f}")


for mode in ("plain", "persistent"):
    for _ in range(3):
        if mode == "plain":
            ctx.run_plain("MM", i.grid, i.args, 0)
        else:
            ctx.run_capped("MM", i.grid, i.args, 0)
    torch.cuda.synchronize()
    read()
    if mode == "plain":
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.run_plain("MM", i.grid, i.args, 0)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
    else:
        ms = ctx.run_capped("MM", i.grid, i.args, 0)
    torch.cuda.synchronize()
    report(f"{mode} {sh}", read(), ms)

#!/usr/bin/env python
"""Device model throughput (a6-a8): one kl_predict batch over every feasible maximal split of
every ordered pair of the ALL-mix kinds (the batch a cold-cache decision issues), timed with
host wall clock around the blocking call (includes the H2D/D2H of the batch) and reported as
candidates/s.  usage: python tools/model_bench.py [reps]"""
import itertools
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from tools.model_error import fits  # noqa: E402


def main(reps):
    profiles, kcfg = bench.load_profiles(os.path.join(ROOT, "profiles", "kl_profile_b200.json"))
    ctx = K.Context(device=0, profiles=profiles, **kcfg)
    smem = torch.cuda.get_device_properties(0).shared_memory_per_multiprocessor
    kinds = G.MIXES["ALL"]
    prof = {k: ctx.get_profile(k) for k in kinds}
    lv = {k: [b for b in range(1, prof[k].bmax + 1) if (b * prof[k].wpb) % 4 == 0] for k in kinds}
    cands = []
    for k1, k2 in itertools.combinations_with_replacement(kinds, 2):
        p1, p2 = prof[k1], prof[k2]
        feas = [(a, b) for a in lv[k1] for b in lv[k2] if fits(p1, a, p2, b, smem) and a * p1.wpb + b * p2.wpb <= 64]
        cands += [(k1, k2, a, b) for a, b in feas
                  if not any((x, y) != (a, b) and x >= a and y >= b for x, y in feas)]
    ctx.predict(cands)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ctx.predict(cands)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    med = ts[len(ts) // 2]
    res = {"candidates": len(cands), "batch_ms_median": med * 1e3, "candidates_per_s": len(cands) / med,
           "reps": reps}
    print(json.dumps(res))
    return res


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 20)

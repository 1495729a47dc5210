#!/usr/bin/env python
"""The paper's OPT comparator: "pre-executes all possible slice
ratios for all combinations to obtain the CP".  Every pair of ALL-mix kinds (same-kind pairs
included) at every maximal occupancy split is co-run on the B200 (kl_run_pair) and its measured
concurrent IPCs, CP and Eq.8 dT become the 'prediction' table that `bench.py --opt` installs
(kl_cache_put, model_frozen) so the same greedy Alg.1 decides from measurements instead of the
Markov model.  Co-run progress is measured inside the window where both kernels are resident
(tools/corun.py, per-block device timestamps).  usage: python tools/opt_table.py [out.json]"""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance  # noqa: E402
from tools.corun import corun, solo_rate, steady_instances  # noqa: E402
from tools.model_error import fits  # noqa: E402

KINDS = G.MIXES["ALL"]


def main(out_path):
    path = os.path.join(ROOT, "profiles", "kl_profile_b200.json")
    profiles, kcfg = bench.load_profiles(path)
    clock = json.load(open(path)).get("clock_mhz_under_ncu", 1965.0) * 1e6
    ctx = K.Context(device=0, profiles=profiles, audit=2, **kcfg)
    props = torch.cuda.get_device_properties(0)
    n_sm, smem_sm = props.multi_processor_count, props.shared_memory_per_multiprocessor
    if os.environ.get("KL_STEADY"):
        # steady state: every kind scaled to a >= 2 ms solo run (tools/corun.py steady_instances)
        calib = json.load(open(path))["measured"]
        a = steady_instances(KINDS, {k: calib[k]["ms_solo"] for k in KINDS})
        b = {k: Instance({"kind": k, "params": a[k].params, "grid_blocks": a[k].grid, "key": a[k].params.get("key")},
                         "cuda", inputs=a[k].inputs) for k in KINDS}
    else:
        data = {k: G.gen(k, "paper") for k in KINDS}
        a = {k: Instance(data[k], "cuda") for k in KINDS}
        b = {k: Instance(data[k], "cuda", inputs=a[k].inputs) for k in KINDS}   # second instance, own outputs
    prof = {k: ctx.get_profile(k) for k in KINDS}
    lv = {k: [x for x in range(1, prof[k].bmax + 1) if (x * prof[k].wpb) % 4 == 0] for k in KINDS}

    def ipc(k, rate):          # blocks per ns -> warp instructions per cycle per virtual SM
        return prof[k].ipb * rate * 1e9 / (clock * 4 * n_sm)

    solo = {k: ipc(k, solo_rate(ctx, k, a[k], lv[k][-1])) for k in KINDS}
    table = []
    for k1, k2 in itertools.combinations_with_replacement(KINDS, 2):
        p1, p2 = prof[k1], prof[k2]
        feas = [(x, y) for x in lv[k1] for y in lv[k2] if fits(p1, x, p2, y, smem_sm)]
        maxi = [(x, y) for x, y in feas if not any((u, v) != (x, y) and u >= x and v >= y for u, v in feas)]
        i1, i2 = a[k1], (b[k2] if k1 == k2 else a[k2])
        for b1, b2 in maxi:
            q1, q2, _ = corun(ctx, k1, i1, b1, k2, i2, b2)
            c1, c2 = ipc(k1, q1), ipc(k2, q2)
            ok = c1 > 0 and c2 > 0
            cp = 1.0 - 1.0 / (c1 / solo[k1] + c2 / solo[k2]) if ok else 0.0
            dT = abs(p1.ipb * b1 / c1 - p2.ipb * b2 / c2) if ok else 0.0
            table.append({"k1": k1, "k2": k2, "b1": b1, "b2": b2, "ipc1": c1, "ipc2": c2, "c": c1 + c2,
                          "solo1": solo[k1], "solo2": solo[k2], "cp": cp, "dT": dT, "status": 0 if ok else 2})
        print(k1, k2, len(maxi), "splits; best measured CP",
              round(max([t["cp"] for t in table if t["k1"] == k1 and t["k2"] == k2] or [0]), 3), flush=True)
    how = ("tools/opt_table.py KL_STEADY=1 (kl_run_pair co-runs, every kind scaled to a >= 2 ms solo run, progress "
           "inside the common window)" if os.environ.get("KL_STEADY") else
           "tools/opt_table.py (kl_run_pair co-runs at paper size, progress inside the common window)")
    json.dump({"solo_ipc": solo, "table": table, "how": how,
               "scale": {k: getattr(a[k], "scale", 1) for k in KINDS}},
              open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "opt_table.json"))

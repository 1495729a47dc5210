#!/usr/bin/env python
"""f2 MC(s) comparator (Fig. randomSchedulingDistribution P:1540-1548): the bench
queue (ALL mix x4, paper sizes) executed s times with random co-schedules -- every decision picks
a uniformly random pending kind pair and maximal slice ratio (kl_config.mc_seed = run number) --
against Kernelet (model-driven, bench configuration) and sequential execution.  Reports the CDF of
the per-queue device time and how many random schedules beat Kernelet.
usage: python tools/mc_cdf.py [s] [out.json]      (needs a GPU)"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance, alloc_outputs, inputs_to_device  # noqa: E402


def main(s, out_path):
    dev = torch.device("cuda", 0)
    profiles, kcfg = bench.load_profiles(os.path.join(ROOT, "profiles", "kl_profile_b200.json"))
    kinds = bench.build_queue(0, 1, 4, "c2")
    data = {k: G.gen(k, "paper") for k in sorted(set(kinds))}
    inputs = {k: inputs_to_device(data[k], dev) for k in data}
    pools, seen, insts = {}, {}, []
    for k in kinds:
        j = seen.get(k, 0)
        seen[k] = j + 1
        if j < 4:
            pools.setdefault(k, []).append(alloc_outputs(k, data[k]["params"], dev))
        insts.append(Instance(data[k], dev, inputs=inputs[k], outputs=pools[k][j % 4]))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def run(ctx, reps):
        ts = []
        for _ in range(reps):
            flush.zero_()
            torch.cuda.synchronize()
            ctx.reset_model_cache()
            ctx.reset_counters()
            ctx.submit_many([(i.kind, i.grid, i.args, n + 1, None) for n, i in enumerate(insts)])
            c = ctx.sync()
            assert c.kernels_done == len(insts)
            ts.append((c.t_end_ns - c.t_start_ns) / 1e6)
        return ts

    counters = torch.zeros(8, dtype=torch.int64, device=dev)
    cfg = dict(kcfg, split_rule=1)
    ctx = K.Context(device=0, profiles=profiles, counters=counters, **cfg)
    run(ctx, 3)
    kern = run(ctx, 10)
    seq = []
    for _ in range(5):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in insts:
            ctx.run_plain(i.kind, i.grid, i.args, 0)
        e1.record()
        e1.synchronize()
        seq.append(e0.elapsed_time(e1))
    ctx.close()
    mc = []
    for seed in range(1, s + 1):
        c = K.Context(device=0, profiles=profiles, counters=counters, mc_seed=seed, **cfg)
        mc += run(c, 1)
        c.close()
        if seed % 100 == 0:
            print(seed, "runs", flush=True)
    k_med = statistics.median(kern)
    mc_sorted = sorted(mc)
    res = {"s": s, "kernelet_ms_median": k_med, "kernelet_ms": kern, "sequential_ms_median": statistics.median(seq),
           "mc_ms_sorted": mc_sorted, "mc_median_ms": statistics.median(mc), "mc_best_ms": mc_sorted[0],
           "mc_worst_ms": mc_sorted[-1], "mc_faster_than_kernelet": sum(1 for x in mc if x < k_med),
           "mc_faster_than_sequential": sum(1 for x in mc if x < statistics.median(seq)),
           "queue": "ALL mix x4 (32 paper-size kernels), device time first block start -> last block end",
           "how": __doc__.split("\n")[0]}
    print(json.dumps({k: v for k, v in res.items() if k not in ("mc_ms_sorted", "kernelet_ms")}))
    json.dump(res, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 200,
         sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "mc_cdf.json"))

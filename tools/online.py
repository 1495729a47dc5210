#!/usr/bin/env python
"""f3: online arrivals (Alg.1 l.2-3 in their true online form; Poisson
arrivals P:1179-1185) with multi-user fairness reporting.

The C5 multi-user queue (16 users, each a Poisson stream from one mix) is replayed at an offered
load rho x the sequential service rate: a resident device arrival clock (kl_arrival_clock, one
thread for the whole run, so arrivals never wait for an SM slot) releases each kernel at its
arrival time by setting its host-mapped ready_flag; Kernelet re-plans on every arrival and every
drain, re-tuning running kernels in place.  The same clock drives two baselines: sequential FIFO
(one stream) and plain multi-stream (4 streams round robin), each launch gated on its flag
(kl_wait_flag) and its completion stamped on the device.  Reported per method: throughput over
the busy period, mean / p95 response time (arrival -> completion), per-user mean slowdown
(response / solo time of the kernel) and Jain's fairness index over users' mean slowdowns.
Kernelet runs twice: the paper's greedy (throughput only), and with the starvation guard
(kl_config.age_limit_us: once the oldest pending kernel waited longer, only co-schedules that
include it are considered).
usage: python tools/online.py [n_kernels] [out.json]      (needs a GPU)"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance, alloc_outputs, inputs_to_device  # noqa: E402


def jain(x):
    x = np.asarray(x, dtype=np.float64)
    return float(x.sum() ** 2 / (len(x) * (x ** 2).sum()))


def summarise(resp_ms, users, kinds, solo, t_first, t_last, n):
    slow = [r / solo[k] for r, k in zip(resp_ms, kinds)]
    per_user = {}
    for u, s in zip(users, slow):
        per_user.setdefault(u, []).append(s)
    um = {u: float(np.mean(v)) for u, v in sorted(per_user.items())}
    return {"kernels_per_s": n / ((t_last - t_first) / 1e3), "busy_ms": t_last - t_first,
            "resp_mean_ms": float(np.mean(resp_ms)), "resp_p95_ms": float(np.percentile(resp_ms, 95)),
            "slowdown_mean": float(np.mean(slow)), "user_mean_slowdown": um, "jain_users": jain(list(um.values()))}


RHOS = [float(x) for x in os.environ.get("RHOS", "0.8,1.0,1.25").split(",")]
AGE_US = int(os.environ.get("AGE_US", "4000"))
LEAD_MS = 30.0   # starvation guard of the kernelet_aged run


def main(n, out_path):
    dev = torch.device("cuda", 0)
    profiles, kcfg = bench.load_profiles(os.path.join(ROOT, "profiles", "kl_profile_b200.json"))
    q = G.multi_user_queue(n, 16, seed=7)
    kinds = [e["kind"] for e in q]
    users = [e["user"] for e in q]
    arr = np.array([e["arrival"] for e in q])
    data = {k: G.gen(k, "paper") for k in sorted(set(kinds))}
    inputs = {k: inputs_to_device(data[k], dev) for k in data}
    pools, seen, insts = {}, {}, []
    for k in kinds:
        j = seen.get(k, 0)
        seen[k] = j + 1
        if j < 4:
            pools.setdefault(k, []).append(alloc_outputs(k, data[k]["params"], dev))
        insts.append(Instance(data[k], dev, inputs=inputs[k], outputs=pools[k][j % 4]))
    counters = torch.zeros(8, dtype=torch.int64, device=dev)
    ctx = K.Context(device=0, profiles=profiles, counters=counters, split_rule=1, **kcfg)
    # solo time per kind (plain launch, full occupancy)
    solo = {}
    for k in data:
        i = next(x for x in insts if x.kind == k)
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.run_plain(k, i.grid, i.args, 0)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        solo[k] = statistics.median(ts)
    seq_ms = sum(solo[k] for k in kinds)
    res = {"n": n, "users": 16, "solo_ms": solo, "sequential_work_ms": seq_ms, "loads": {}}
    arr_stream = torch.cuda.Stream(device=dev)
    for rho in RHOS:
        # arrival times scaled so that the offered load is rho x the sequential service rate
        span = seq_ms / rho
        t = (arr - arr[0]) / max(arr[-1] - arr[0], 1e-12) * span * 1e6 if n > 1 else np.zeros(1)
        gaps = np.diff(np.concatenate([[0.0], t])).astype(np.int64)
        # lead-in: every method has enqueued all its work before the first arrival
        gaps[0] += int(LEAD_MS * 1e6)
        gaps_d = torch.tensor(gaps, dtype=torch.int64, device=dev)
        out = {}

        def clock():
            """Fresh flags (host-mapped) and stamps; start the resident arrival clock."""
            flags = torch.zeros(n, dtype=torch.int32).pin_memory()
            stamps = torch.zeros(n, dtype=torch.int64, device=dev)
            return flags, stamps

        # --- Kernelet: the paper's greedy, and with the starvation guard (serving extension)
        for name, age in (("kernelet", 0), ("kernelet_aged", AGE_US)):
            ctx.close()
            ctx = K.Context(device=0, profiles=profiles, counters=counters, split_rule=1, age_limit_us=age, **kcfg)
            flags, stamps = clock()
            torch.cuda.synchronize()
            n0 = len(ctx.trace())
            s0 = ctx.stats()
            ids = ctx.submit_many([(x.kind, x.grid, x.args, m + 1, None, flags.data_ptr() + 4 * m)
                                   for m, x in enumerate(insts)])
            ctx.arrival_clock(arr_stream, gaps_d.data_ptr(), stamps.data_ptr(), flags.data_ptr(), n)
            ctx.sync()
            torch.cuda.synchronize()
            s1 = ctx.stats()
            tr = ctx.trace()[n0:]
            done = {t_.id: t_.t1_ns for t_ in tr if t_.exhausted}
            st = stamps.cpu().numpy()
            resp = [(done[kid] - st[m]) / 1e6 for m, kid in enumerate(ids)]
            out[name] = summarise(resp, users, kinds, solo, st[0] / 1e6, max(done.values()) / 1e6, n)
            out[name]["stats"] = {f: getattr(s1, f) - getattr(s0, f) for f, _ in K.Stats._fields_}
            out[name]["age_limit_us"] = age
            first = {}
            for t_ in tr:
                if t_.admitted:
                    first[t_.id] = min(first.get(t_.id, 1 << 62), t_.t0_ns)
            z = int(st[0])
            out[name]["per_kernel"] = [{"kind": kinds[m], "user": users[m], "arrive_us": (int(st[m]) - z) / 1e3,
                                        "start_us": (first.get(kid, z) - z) / 1e3, "done_us": (done[kid] - z) / 1e3}
                                       for m, kid in enumerate(ids)]
        # --- sequential FIFO and plain multi-stream (4 streams): each launch gated on its arrival
        # flag (kl_wait_flag), completion stamped on the device after it
        for name, nstreams in (("sequential", 1), ("multistream4", 4)):
            streams = [torch.cuda.Stream(device=dev) for _ in range(nstreams)]
            flags, stamps = clock()
            dstamp = torch.zeros(n, dtype=torch.int64, device=dev)
            torch.cuda.synchronize()
            for m, x in enumerate(insts):
                s = streams[m % nstreams]
                ctx.wait_flag(s, flags.data_ptr() + 4 * m, None)
                ctx.run_plain(x.kind, x.grid, x.args, s)
                ctx.wait_flag(s, None, dstamp.data_ptr() + 8 * m)
            ctx.arrival_clock(arr_stream, gaps_d.data_ptr(), stamps.data_ptr(), flags.data_ptr(), n)
            torch.cuda.synchronize()
            st = stamps.cpu().numpy()
            dn = dstamp.cpu().numpy()
            resp = [(int(dn[m]) - int(st[m])) / 1e6 for m in range(n)]
            out[name] = summarise(resp, users, kinds, solo, st[0] / 1e6, dn.max() / 1e6, n)
        res["loads"][str(rho)] = out
        print(rho, {m: {f: round(float(v[f]), 3) for f in ("kernels_per_s", "resp_mean_ms", "resp_p95_ms",
                                                            "slowdown_mean", "jain_users")} for m, v in out.items()},
              flush=True)
    ctx.close()
    json.dump(res, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 320,
         sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "online.json"))

#!/usr/bin/env python
"""How far is Alg.1's greedy from the best pairwise plan on a big queue?  A fluid study over the
measured pair table (`tools/opt_table.py`: every ALL-mix pair at every maximal split co-run on
the B200, rates r_k = cIPC_k / IPC_k^solo) and the Markov model's predictions for the same
candidates.  For a queue with solo work W_k per kind (ms, from the bench's per-kind solo times):
  * LP(measured): min sum t_c s.t. sum_c r_{c,k} t_c = W_k, t >= 0 -- the optimal fluid makespan
    of pairwise co-schedules (plus solo runs) with measured rates;
  * LP(model) evaluated on measured rates: the plan an LP planner on the model's predictions
    would follow (its time shares), replayed with the measured rates, leftovers run solo;
  * greedy(model / measured): the fluid Alg.1 -- at each point the max-CP candidate among the
    pending kinds (model or measured CP), run until one of its kinds is done -- replayed with the
    measured rates.
CPU post-processing of two JSON files; the model predictions are fetched on the GPU box
(`python tools/lp_study.py predict OUT.json`), the study runs anywhere.
usage: python tools/lp_study.py predict gpurun_out/r02_model_preds.json      (GPU)
       python tools/lp_study.py study OPT_TABLE.json PREDS.json BENCH.json [OUT.json]"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def predict(out_path):
    import bench
    import paper_1303_5164_b200 as K
    path = os.path.join(ROOT, "profiles", "kl_profile_b200.json")
    profiles, kcfg = bench.load_profiles(path)
    ctx = K.Context(device=0, profiles=profiles, **kcfg)
    opt = json.load(open(os.path.join(ROOT, "profiles", "r02_opt_table.json")))
    cands = [(t["k1"], t["k2"], t["b1"], t["b2"]) for t in opt["table"]]
    pr = ctx.predict(cands)
    out = [{"k1": c[0], "k2": c[1], "b1": c[2], "b2": c[3], "ipc1": p.ipc1, "ipc2": p.ipc2, "solo1": p.solo1,
            "solo2": p.solo2, "cp": p.cp, "status": p.status} for c, p in zip(cands, pr)]
    json.dump(out, open(out_path, "w"), indent=1)


def rates(rows, solo=None):
    """(k1, k2, b1, b2) -> (r1, r2): progress rates relative to solo."""
    out = {}
    for t in rows:
        if t.get("status", 0) != 0:
            continue
        s1 = solo[t["k1"]] if solo else t["solo1"]
        s2 = solo[t["k2"]] if solo else t["solo2"]
        out[(t["k1"], t["k2"], t["b1"], t["b2"])] = (t["ipc1"] / s1, t["ipc2"] / s2)
    return out


def lp(W, R):
    import numpy as np
    from scipy.optimize import linprog
    kinds = sorted(W)
    cols, keys = [], []
    for key, (r1, r2) in R.items():
        k1, k2 = key[0], key[1]
        if k1 not in W or k2 not in W:
            continue
        col = np.zeros(len(kinds))
        col[kinds.index(k1)] += r1
        col[kinds.index(k2)] += r2
        cols.append(col)
        keys.append(key)
    for k in kinds:
        col = np.zeros(len(kinds))
        col[kinds.index(k)] = 1.0
        cols.append(col)
        keys.append((k, "solo"))
    M = np.array(cols).T
    res = linprog(np.ones(M.shape[1]), A_eq=M, b_eq=[W[k] for k in kinds], bounds=(0, None), method="highs")
    return res.fun, {keys[i]: float(x) for i, x in enumerate(res.x) if x > 1e-9}


def replay(plan, W, Rm):
    """Run plan's time shares with the measured rates; leftover work solo."""
    rem = dict(W)
    t = 0.0
    for key, dt in sorted(plan.items(), key=lambda kv: -kv[1]):
        if key[1] == "solo":
            continue
        r1, r2 = Rm.get(key, (0.0, 0.0))
        k1, k2 = key[0], key[1]
        # run for dt or until one kind is done
        d = dt
        if r1 > 0:
            d = min(d, rem[k1] / r1)
        if r2 > 0:
            d = min(d, rem[k2] / r2)
        rem[k1] -= r1 * d
        rem[k2] -= r2 * d
        t += d
    return t + sum(max(0.0, v) for v in rem.values())


def greedy(W, Rdec, Rmeas, cp_of):
    rem = {k: v for k, v in W.items() if v > 0}
    t = 0.0
    while rem:
        best = None
        for key, (r1, r2) in Rdec.items():
            k1, k2 = key[0], key[1]
            if k1 == k2 or k1 not in rem or k2 not in rem:
                continue
            cp = cp_of(key)
            if best is None or cp > best[0]:
                best = (cp, key)
        if best is None or best[0] <= 0:
            k = next(iter(rem))
            t += rem.pop(k)
            continue
        key = best[1]
        r1, r2 = Rmeas[key]
        k1, k2 = key[0], key[1]
        d = min(rem[k1] / r1 if r1 > 0 else 1e18, rem[k2] / r2 if r2 > 0 else 1e18)
        rem[k1] -= r1 * d
        rem[k2] -= r2 * d
        t += d
        for k in (k1, k2):
            if rem[k] <= 1e-9 * W[k]:
                rem.pop(k)
    return t


def study(opt_path, preds_path, bench_path, out_path=None):
    import bench
    opt = json.load(open(opt_path))
    preds = json.load(open(preds_path))
    b = json.load(open(bench_path))
    pk = {k: v["ms"] for k, v in b["roofline_all"].items()}
    cnt = collections.Counter(bench.global_queue("c5", 4, 1))
    W = {k: cnt[k] * pk[k] for k in cnt}
    Rm = rates(opt["table"], opt["solo_ipc"])
    Rp = rates(preds)
    cp_meas = {k: next(t["cp"] for t in opt["table"] if (t["k1"], t["k2"], t["b1"], t["b2"]) == k) for k in Rm}
    cp_pred = {(t["k1"], t["k2"], t["b1"], t["b2"]): t["cp"] for t in preds if t["status"] == 0}
    lp_m, plan_m = lp(W, Rm)
    lp_p, plan_p = lp(W, {k: v for k, v in Rp.items() if k in Rm})
    res = {"queue": "C5 (10,000 kernels), solo work per kind (ms)", "W_ms": W, "sequential_ms": sum(W.values()),
           "lp_measured_ms": lp_m, "lp_measured_plan": {"|".join(map(str, k)): v for k, v in plan_m.items()},
           "lp_model_plan_replayed_ms": replay(plan_p, W, Rm),
           "greedy_model_cp_replayed_ms": greedy(W, {k: v for k, v in Rp.items() if k in Rm}, Rm,
                                                 lambda k: cp_pred.get(k, -1)),
           "greedy_measured_cp_ms": greedy(W, Rm, Rm, lambda k: cp_meas[k]),
           "bench_measured_ms": b.get("ms_per_step")}
    s = json.dumps(res, indent=1)
    print(s)
    if out_path:
        open(out_path, "w").write(s)


if __name__ == "__main__":
    if sys.argv[1] == "predict":
        predict(sys.argv[2])
    else:
        study(*sys.argv[2:])

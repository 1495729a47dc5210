#!/usr/bin/env python
"""Fit MM's effective model inputs to its measured co-runs (reading R20: the asynchronous
TMA/tcgen05 kernel does not fit the two-state warp model, and its solo occupancy sweep has a single
level -- one 196-KB block per SM -- so the solo fit of tools/calibrate.py cannot see how it shares
an SM).  Grid search over MM's (Rm, r, pipe ceiling pi on a pipe of its own) with the device model
(kl_predict), minimising the mean |CP_pred - CP_meas| over every measured MM pair and maximal
split of the OPT table (profiles/r01_opt_table.json, tools/opt_table.py) plus the relative error of
MM's solo IPC.  Writes the profile with the fitted MM entry.

usage: python tools/fit_mm_corun.py OUT_PROFILE.json      (needs a GPU)"""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402

PIPE_TENSOR = 4   # a pipe id no other kind uses: MM's ceiling only bounds MM's own rounds


def main(out_path: str) -> None:
    prof_path = os.path.join(ROOT, "profiles", "kl_profile_b200.json")
    raw = json.load(open(prof_path))
    profiles, kcfg = bench.load_profiles(prof_path)
    opt = json.load(open(os.path.join(ROOT, "profiles", "r01_opt_table.json")))
    rows = [r for r in opt["table"] if r["status"] == 0 and "MM" in (r["k1"], r["k2"]) and r["k1"] != r["k2"]]
    solo_meas = opt["solo_ipc"]["MM"]
    ctx = K.Context(device=0, profiles=profiles, **kcfg)
    base = dict(raw["profiles"]["MM"])
    cands = [(r["k1"], r["k2"], r["b1"], r["b2"]) for r in rows]

    def score(p):
        ctx.set_profile("MM", p)
        ctx.reset_model_cache()
        pr = ctx.predict(cands + [("MM", "MM", 1, 0)])
        ok = [(q, r) for q, r in zip(pr[:-1], rows) if q.status == 0]
        if len(ok) < len(rows) or pr[-1].status != 0:
            return None
        e_cp = sum(abs(q.cp - r["cp"]) for q, r in ok) / len(ok)
        e_solo = abs(pr[-1].ipc1 - solo_meas) / solo_meas
        return e_cp + 0.5 * e_solo, e_cp, e_solo

    results = []
    for rm, r, pi in itertools.product([0.01, 0.02, 0.043, 0.08, 0.15, 0.3, 0.5],
                                       [1.0, 4.0, 16.0, 64.0],
                                       [1.0, 0.5, 0.2, 0.1, 0.05, 0.02]):
        p = dict(base, rm=rm, r=r, ipc_max=pi, pipe=PIPE_TENSOR if pi < 1.0 else 0)
        s = score(p)
        if s:
            results.append((s, {"rm": rm, "r": r, "ipc_max": pi, "pipe": p["pipe"]}))
    results.sort(key=lambda x: x[0][0])
    s0 = score(base)
    best_s, best = results[0]
    print("profiled/solo-fit MM:", {k: base[k] for k in ("rm", "r", "ipc_max", "pipe")},
          "objective %.4f  mean |dCP| %.4f  solo rel err %.4f" % s0)
    print("co-run fit MM:      ", best, "objective %.4f  mean |dCP| %.4f  solo rel err %.4f" % best_s)
    for s, q in results[1:6]:
        print("   next:", q, "%.4f %.4f %.4f" % s)
    out = json.loads(json.dumps(raw))
    out["profiles"]["MM"].update(best)
    out["profiles"]["MM"]["corun_fit"] = {"objective": best_s[0], "mean_abs_dcp": best_s[1], "solo_rel_err": best_s[2],
                                          "before": {"objective": s0[0], "mean_abs_dcp": s0[1], "solo_rel_err": s0[2]},
                                          "n_rows": len(rows), "how": __doc__.split("\n\n")[0]}
    with open(out_path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", out_path)


if __name__ == "__main__":
    main(sys.argv[1])

#!/usr/bin/env python
"""f1 study (the paper's "Model Optimizations" experiment): predicted vs measured solo
IPC per virtual SM of the kernels with uncoalesced accesses (PC, SPMV) at every occupancy level,
and of their co-runs (config C3 cases in profiles/r01_model_error.json), under
  (a) the two-state model with every memory instruction treated as coalesced (r = 4 sectors),
  (b) the two-state model with the profiled mean sectors per request,
  (c) the three-state model (model_states = 3): uc = (mean - 4)/(32 - 4) of the memory
      instructions uncoalesced at 32 sectors, the rest coalesced at 4 (reading R27),
all from the profiled (not fitted) Rm and the calibrated L0/B, evaluated by the device model
(kl_predict; solo queries b2 = 0).  Measured IPCs come from the committed calibration
(profiles/kl_profile_b200.json: occupancy sweeps) and C3 co-runs.
usage: python tools/model3_study.py [out.json]      (needs a GPU)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1303_5164_b200 as K  # noqa: E402

COAL, UNCOAL = 4.0, 32.0      # sectors per warp request: 32 lanes x 4 B, and one sector per lane


def variants(calib):
    out = {}
    for name in ("two_coalesced", "two_mean", "three"):
        profs = {}
        for k, p in calib["profiles"].items():
            raw = calib["measured"].get(k, {}).get("raw", {})
            req = raw.get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")
            sec = raw.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")
            mean = sec / req if req else p.get("r_profiled", p["r"])
            q = {f: p[f] for f in ("rm", "r", "ipb", "pur", "mur", "m_min", "ipc_max", "pipe") if f in p}
            q["rm"] = p.get("rm_profiled", p["rm"])
            if name == "two_coalesced":
                q.update(r=COAL, uc=0.0, ru=COAL)
            elif name == "two_mean":
                q.update(r=mean, uc=0.0, ru=mean)
            else:
                uc = min(1.0, max(0.0, (mean - COAL) / (UNCOAL - COAL)))
                q.update(r=COAL, uc=uc, ru=UNCOAL)
            profs[k] = q
        out[name] = profs
    return out


def main(out_path):
    calib = json.load(open(os.path.join(ROOT, "profiles", "kl_profile_b200.json")))
    cfg = calib["config"]
    me = json.load(open(os.path.join(ROOT, "profiles", "r01_model_error.json")))
    res = {"solo": {}, "pairs": {}, "how": __doc__.split("\n")[0]}
    for name, profs in variants(calib).items():
        ctx = K.Context(device=0, profiles=profs, model_states=3 if name == "three" else 2, **cfg)
        solo_err = {}
        for k in ("PC", "SPMV", "ST", "BS", "TEA", "SAD", "MRIQ"):
            meas = calib["measured"].get(k, {}).get("ipc_meas", {})
            p = ctx.get_profile(k)
            caps = [int(c) for c in meas if (int(c) * p.wpb) % 4 == 0]
            preds = ctx.predict([(k, k, c, 0) for c in caps])
            rows = [(c, meas[str(c)], pr.ipc1) for c, pr in zip(caps, preds) if pr.status == 0]
            solo_err[k] = {"mean_abs_err": float(np.mean([abs(a - b) for _, a, b in rows])) if rows else None,
                           "points": [{"cap": c, "meas": a, "pred": b} for c, a, b in rows]}
        res["solo"][name] = solo_err
        # co-runs involving PC / SPMV (C3 cases, measured cIPC per vSM)
        cases = [c for c in me["cases"] if "PC" in (c["k1"], c["k2"]) or "SPMV" in (c["k1"], c["k2"])]
        preds = ctx.predict([(c["k1"], c["k2"], c["b1"], c["b2"]) for c in cases])
        errs = []
        for c, pr in zip(cases, preds):
            if pr.status == 0:
                errs += [abs(pr.ipc1 - c["meas"]["ipc1"]), abs(pr.ipc2 - c["meas"]["ipc2"])]
        res["pairs"][name] = {"mean_abs_cipc_err": float(np.mean(errs)) if errs else None, "n": len(errs) // 2}
        ctx.close()
        print(name, {k: (round(v["mean_abs_err"], 4) if v["mean_abs_err"] is not None else None)
                     for k, v in solo_err.items()}, "pairs", res["pairs"][name], flush=True)
    json.dump(res, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "model3_study.json"))

#!/usr/bin/env python
"""Config C3 / paper E4, E5, E7 analogs: the Markov model's predictions against measured
co-execution on the B200 (GPU box).

For every pair of the eight ALL-mix kernels at paper size and three slice ratios -- the one the
model picks by argmax CP (split_rule 1), the balanced ratio of Eq.8 (split_rule 0) and the most
even 1:1 warp split -- both kernels run concurrently through the slice launcher (kl_run_pair)
until the first runs out of thread blocks.  Measured concurrent IPC per virtual SM:
    cIPC_k = I_k * blocks_executed_k / (window_k * f * 4 * n_SM)
and measured CP = 1 - 1/(sum cIPC_k / IPC_k^solo) with the solo IPC measured at b_max; each kernel's
progress is counted inside the window where both are resident (tools/corun.py, per-block device
timestamps), so neither the ramp-up nor the survivor's solo tail enters the co-run rates.  Reports the paper's metric, the average absolute IPC error per virtual SM
(0.08 on C2050), and the CP error.
KL_C3_SYNTH=1 adds the synthetic streaming kernel (4 FMAs per element), i.e. config C3's
tensor-core MM vs streaming pair among 8 more.
usage: python tools/model_error.py [out.json]      (KL_PROFILE=path: another calibration file)"""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import kl_inputs as G  # noqa: E402
import paper_1303_5164_b200 as K  # noqa: E402
from paper_1303_5164_b200.workload import Instance  # noqa: E402
from tools.corun import corun, solo_rate, steady_instances  # noqa: E402

KINDS = G.MIXES["ALL"] + (["SYNTH"] if os.environ.get("KL_C3_SYNTH") else [])   # C3: + the streaming kernel


def fits(p1, b1, p2, b2, sm):
    w = b1 * p1.wpb + b2 * p2.wpb
    regs = sum(b * pr.wpb * ((pr.regs * 32 + 255) // 256 * 256) for pr, b in ((p1, b1), (p2, b2)))
    smem = sum(b * (pr.smem + 1024) for pr, b in ((p1, b1), (p2, b2)))
    tmem = b1 * p1.tmem + b2 * p2.tmem
    return w <= 64 and b1 + b2 <= 32 and regs <= 65536 and smem <= sm and tmem <= 512


def main(out_path):
    path = os.environ.get("KL_PROFILE") or os.path.join(ROOT, "profiles", "kl_profile_b200.json")
    profiles, kcfg = bench.load_profiles(path)
    calib = json.load(open(path))
    clock = calib.get("clock_mhz_under_ncu", 1965.0) * 1e6
    ctx = K.Context(device=0, profiles=profiles, audit=2, **kcfg)
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    smem_sm = torch.cuda.get_device_properties(0).shared_memory_per_multiprocessor
    if os.environ.get("KL_STEADY"):     # every kind scaled to a >= 2 ms solo run (tools/corun.py)
        insts = steady_instances(KINDS, {k: calib["measured"][k]["ms_solo"] for k in KINDS})
    else:
        insts = {k: Instance(G.gen(k, "paper"), "cuda") for k in KINDS}
    prof = {k: ctx.get_profile(k) for k in KINDS}
    lv = {k: [b for b in range(1, prof[k].bmax + 1) if (b * prof[k].wpb) % 4 == 0] for k in KINDS}
    solo_b = {k: lv[k][-1] for k in KINDS}

    def ipc_of(k, rate):       # blocks per ns -> warp instructions per cycle per virtual SM
        return prof[k].ipb * rate * 1e9 / (clock * 4 * n_sm)

    solo = {k: ipc_of(k, solo_rate(ctx, k, insts[k], solo_b[k])) for k in KINDS}
    cases = []
    for k1, k2 in itertools.combinations(KINDS, 2):
        p1, p2 = prof[k1], prof[k2]
        feas = [(a, b) for a in lv[k1] for b in lv[k2] if fits(p1, a, p2, b, smem_sm)]
        maxi = [(a, b) for a, b in feas if not any((x, y) != (a, b) and x >= a and y >= b for x, y in feas)]
        if not maxi:
            continue
        preds = ctx.predict([(k1, k2, a, b) for a, b in maxi])
        ok = [(s, p) for s, p in zip(maxi, preds) if p.status == 0]
        if not ok:
            continue
        pick = {"argmax_cp": max(ok, key=lambda t: t[1].cp)[0],
                "balanced_dT": min(ok, key=lambda t: t[1].dT)[0],
                "one_to_one": min(ok, key=lambda t: abs(t[0][0] * p1.wpb - t[0][1] * p2.wpb))[0]}
        for rule, (b1, b2) in pick.items():
            pr = dict(ok)[(b1, b2)]
            q1, q2, wns = corun(ctx, k1, insts[k1], b1, k2, insts[k2], b2)
            c1, c2 = ipc_of(k1, q1), ipc_of(k2, q2)
            if not (c1 > 0 and c2 > 0):     # the two never ran at the same time (no window)
                print(k1, k2, b1, b2, rule, "no co-run window", flush=True)
                continue
            cp_meas = 1.0 - 1.0 / (c1 / solo[k1] + c2 / solo[k2])
            cases.append({"k1": k1, "k2": k2, "b1": b1, "b2": b2, "rule": rule,
                          "pred": {"ipc1": pr.ipc1, "ipc2": pr.ipc2, "cp": pr.cp},
                          "meas": {"ipc1": c1, "ipc2": c2, "cp": cp_meas},
                          "window_ms": wns / 1e6})
            print(k1, k2, b1, b2, rule, "pred", round(pr.ipc1, 3), round(pr.ipc2, 3), round(pr.cp, 3),
                  "meas", round(c1, 3), round(c2, 3), round(cp_meas, 3), flush=True)
    e_ipc = [abs(c["pred"][f] - c["meas"][f]) for c in cases for f in ("ipc1", "ipc2")]
    e_cp = [abs(c["pred"]["cp"] - c["meas"]["cp"]) for c in cases]
    solo_err = {k: calib["measured"].get(k, {}).get("fit", {}).get("rmse") for k in KINDS}
    summary = {"steady": bool(os.environ.get("KL_STEADY")),
               "mean_abs_cipc_err_per_vsm": float(np.mean(e_ipc)), "max_abs_cipc_err": float(np.max(e_ipc)),
               "mean_abs_cp_err": float(np.mean(e_cp)), "n_cases": len(cases),
               "solo_ipc_measured": solo, "solo_fit_rmse": solo_err,
               "paper": "C2050 average absolute IPC error 0.08 (peak 1), GTX680 0.21 (peak 8), P:1299-1303"}
    print(json.dumps(summary, indent=1))
    json.dump({"summary": summary, "cases": cases}, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "model_error.json"))

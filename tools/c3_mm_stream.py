#!/usr/bin/env python
"""Config C3: the tensor-core MM (CTA pairs, tcgen05) against the synthetic
streaming kernel over MM's occupancy levels -- its TMA ring depths S in {2, 3, 4, 6}
(kl_config.mm_stages) -- and the streaming kernel's memory-instruction ratio Rm (c dependent FMAs
per loaded float4: c = 4, 2, 1, 0 give Rm ~ 0.06, 0.10, 0.16, 0.42), at two slice ratios: the
maximal split (MM 1 block per SM, the streamer at its largest feasible level) and the 1:1 warp
split (one 8-warp streamer block beside MM's 8 warps).

Per case: measured co-run rates inside the common window (tools/corun.py, device per-block
timestamps), measured CP = 1 - 1/(r_MM + r_SYNTH) with r = co-run rate / solo rate (MM's solo rate
at the same ring depth; R20: MM's "IPC" is its tile-progress rate), and the model's prediction for
the same candidate.  The streamer's model inputs at each c follow from its calibration at c = 4: I
per block from the instruction count ratio, and the effective stall rate = the profiled Rm divided
by the memory-level parallelism the calibration fitted (profiled / effective Rm at c = 4).
usage: python tools/c3_mm_stream.py [out.json]      (needs a GPU)"""
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
from tools.corun import corun, solo_rate  # noqa: E402

STAGES = [2, 3, 4, 6]
FMAS = [4, 2, 1, 0]


def main(out_path):
    path = os.path.join(ROOT, "profiles", "kl_profile_b200.json")
    profiles, kcfg = bench.load_profiles(path)
    calib = json.load(open(path))
    clock = calib.get("clock_mhz_under_ncu", 1965.0) * 1e6
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    mm = Instance(G.gen("MM", "paper"), "cuda")
    base = calib["profiles"]["SYNTH"]
    # instructions per loaded float4 of the streamer: 1 load + 4c FFMA + loop overhead; the
    # overhead follows from the profiled Rm at c = 4 (Rm = 1 / (1 + 16 + ovh))
    ovh = 1.0 / base["rm_profiled"] - 17.0
    out = {"stages": STAGES, "fmas": FMAS, "cases": [], "solo": {}}
    synth = {}
    for c in FMAS:
        d = G.gen("SYNTH", "paper", fmas=c)
        synth[c] = Instance(d, "cuda")
    for S in STAGES:
        ctx = K.Context(device=0, profiles=profiles, audit=2, mm_stages=S, **kcfg)
        pm = ctx.get_profile("MM")
        r_mm = solo_rate(ctx, "MM", mm, 0)
        out["solo"][f"MM{S}"] = {"blocks_per_us": r_mm * 1e3, "ms": mm.grid / r_mm / 1e6}
        for c in FMAS:
            i = synth[c]
            rm_prof = 1.0 / (1.0 + 4 * c + ovh)
            ipb = base["ipb"] * (1.0 + 4 * c + ovh) / (17.0 + ovh)
            q = dict(profiles["SYNTH"], ipb=ipb, rm=base["rm"] * rm_prof / base["rm_profiled"])
            ctx.set_profile("SYNTH", q)
            ps = ctx.get_profile("SYNTH")
            r_s = solo_rate(ctx, "SYNTH", i, 0)
            b_max = next(b for b in range(ps.bmax, 0, -1)
                         if (b * ps.wpb + pm.wpb) <= 64 and
                         b * ps.wpb * ((ps.regs * 32 + 255) // 256 * 256) + pm.wpb * ((pm.regs * 32 + 255) // 256 * 256) <= 65536)
            for split, b2 in (("maximal", b_max), ("one_to_one", max(1, pm.wpb // ps.wpb))):
                q1, q2, wns = corun(ctx, "MM", mm, 1, "SYNTH", i, b2)
                if not (q1 > 0 and q2 > 0):
                    continue
                rr1, rr2 = q1 / r_mm, q2 / r_s
                pr = ctx.predict([("MM", "SYNTH", 1, b2)])[0]
                case = {"stages": S, "fmas": c, "rm": rm_prof, "split": [1, b2], "split_rule": split,
                        "meas": {"r_mm": rr1, "r_synth": rr2, "cp": 1.0 - 1.0 / (rr1 + rr2)},
                        "pred": {"r_mm": pr.ipc1 / pr.solo1 if pr.solo1 else None,
                                 "r_synth": pr.ipc2 / pr.solo2 if pr.solo2 else None, "cp": pr.cp},
                        "window_ms": wns / 1e6,
                        "mm_variant": next(t.variant for t in ctx.trace()[-2:] if t.kind == K.KIND_ID["MM"])}
                out["cases"].append(case)
                print(json.dumps(case), flush=True)
        ctx.close()
    e = [abs(c["pred"]["cp"] - c["meas"]["cp"]) for c in out["cases"]]
    out["summary"] = {"mean_abs_cp_err": float(np.mean(e)) if e else None, "n": len(e),
                      "mm_solo_us_by_stages": {k: round(v["ms"] * 1e3, 1) for k, v in out["solo"].items()}}
    print(json.dumps(out["summary"], indent=1))
    json.dump(out, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "c3_mm_stream.json"))

#!/usr/bin/env python
"""Launch-order / occupancy study of MRIQ (the MUFU-bound kind that carries half of C5's work) and
its partners, in steady state (every kind scaled so its solo run takes >= 2 ms, MRIQ >= 8 ms so it
outlives the partner).  For every partner X and MRIQ cap m in 1..5, X at its maximal fit beside
MRIQ; both launch orders (MRIQ first = the C5 operating point, where MRIQ is resident when its
partners join; X first).  Rates are normalised by the kind's solo rate at its own b_max, so a pair's
r1 + r2 is its combined progress (> 1: co-running pays).
usage: python tools/mriq_partner.py [out.json] [partners=PC,SAD,ST,BS,TEA,SPMV]   (needs a GPU)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1303_5164_b200 as K  # noqa: E402
from tools.corun import corun, solo_rate, steady_instances  # noqa: E402

out_path = sys.argv[1] if len(sys.argv) > 1 else None
partners = (sys.argv[2] if len(sys.argv) > 2 else "PC,SAD,ST,BS,TEA,SPMV").split(",")
prof = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                   "kl_profile_b200.json")))
solo_ms = {k: float(v["ms_solo"]) for k, v in prof["measured"].items() if "ms_solo" in v}
ctx = K.Context(device=0, audit=2)
insts = steady_instances(partners, solo_ms, 2.0)
insts.update(steady_instances(["MRIQ"], solo_ms, 8.0))
P = {k: ctx.get_profile(k) for k in insts}


def fit(m, p):
    """Largest cap of partner p beside m MRIQ blocks per SM (warps, registers, shared memory, blocks)."""
    q = P["MRIQ"]
    best = 0
    for c in range(1, p.bmax + 1):
        warps = m * q.wpb + c * p.wpb
        regs = m * q.wpb * 32 * q.regs + c * p.wpb * 32 * p.regs
        smem = m * (q.smem + 1024) + c * (p.smem + 1024)
        if warps <= 64 and regs <= 65536 and smem <= 233472 and m + c <= 32:
            best = c
    return best


solo = {}
for k, i in insts.items():
    solo[k] = solo_rate(ctx, k, i, 0)
print("solo blocks/us", {k: round(v * 1e3, 3) for k, v in solo.items()}, flush=True)
rows = []
for x in partners:
    for m in range(1, 6):
        c = fit(m, P[x])
        if c == 0:
            continue
        for order in ("MRIQ_first", "X_first"):
            if order == "MRIQ_first":
                r_q, r_x, w = corun(ctx, "MRIQ", insts["MRIQ"], m, x, insts[x], c)
            else:
                r_x, r_q, w = corun(ctx, x, insts[x], c, "MRIQ", insts["MRIQ"], m)
            row = dict(partner=x, mriq_cap=m, partner_cap=c, order=order, r_mriq=r_q / solo["MRIQ"],
                       r_partner=r_x / solo[x], window_us=w / 1e3)
            row["sum"] = row["r_mriq"] + row["r_partner"]
            rows.append(row)
            print(f"{x:5s} m={m} c={c:2d} {order:10s} MRIQ {row['r_mriq']:.2f}  {x} {row['r_partner']:.2f}  "
                  f"sum {row['sum']:.2f}  window {row['window_us']:.0f} us", flush=True)
torch.cuda.synchronize()
if out_path:
    json.dump(dict(how=__doc__, solo_blocks_per_ns=solo, scale={k: i.scale for k, i in insts.items()}, rows=rows),
              open(out_path, "w"), indent=1)

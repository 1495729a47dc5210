#!/usr/bin/env python
"""f4: PUR/MUR pruning recalibrated for B200 (tb:pruningTableC2050 P:1497-1531).

Inputs are measured artefacts only: each kind's PUR and MUR from the ncu calibration
(profiles/kl_profile_b200.json; R15/R23 normalisation) and the best measured co-scheduling profit
of every pair of the ALL-mix kinds over its maximal slice ratios (profiles/r01_opt_table.json,
kl_run_pair co-runs at paper size).  Reports
  * the correlation of the best measured CP with |dPUR| and |dMUR| (the paper's Fig. pur_mur
    premise: complementary kernels co-schedule better),
  * the B200 pruning table -- pairs of C(8,2) = 28 pruned under the AND rule (R9) for the
    paper's alpha grid -- with, per cell, how many profitable pairs (best measured CP >= 0.15)
    it would prune,
  * the recalibrated defaults: the cell with the most pairs pruned that prunes no profitable
    pair, ties to the smaller thresholds,
  * the p% rule per kind (minimum slice in waves, from the calibration's stop-and-relaunch sweep).
Runs on the CPU.  usage: python tools/pruning_study.py [out.json]"""
import itertools
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KINDS = ["PC", "SAD", "SPMV", "ST", "MM", "MRIQ", "BS", "TEA"]
AP = [0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0]
AM = [0.015, 0.03, 0.045, 0.06, 0.075, 0.09, 0.105, 0.12, 0.135, 0.15]
PROFITABLE = 0.15


def spearman(x, y):
    rx = np.argsort(np.argsort(x)).astype(float)
    ry = np.argsort(np.argsort(y)).astype(float)
    return float(np.corrcoef(rx, ry)[0, 1])


def main(out_path):
    calib = json.load(open(os.path.join(ROOT, "profiles", "kl_profile_b200.json")))
    tab = json.load(open(os.path.join(ROOT, "profiles", "r01_opt_table.json")))["table"]
    pur = {k: calib["profiles"][k]["pur"] for k in KINDS}
    mur = {k: calib["profiles"][k]["mur"] for k in KINDS}
    best = {}
    for t in tab:
        if t["status"] != 0 or t["k1"] == t["k2"]:
            continue
        key = tuple(sorted((t["k1"], t["k2"])))
        best[key] = max(best.get(key, -9.0), t["cp"])
    pairs = [p for p in itertools.combinations(sorted(KINDS), 2) if p in best]
    dp = np.array([abs(pur[a] - pur[b]) for a, b in pairs])
    dm = np.array([abs(mur[a] - mur[b]) for a, b in pairs])
    cp = np.array([best[p] for p in pairs])
    res = {"pur": pur, "mur": mur, "best_measured_cp": {f"{a}+{b}": best[(a, b)] for a, b in pairs},
           "correlation": {"pearson_cp_dpur": float(np.corrcoef(cp, dp)[0, 1]),
                           "pearson_cp_dmur": float(np.corrcoef(cp, dm)[0, 1]),
                           "spearman_cp_dpur": spearman(cp, dp), "spearman_cp_dmur": spearman(cp, dm),
                           "pearson_cp_dpur_plus_dmur": float(np.corrcoef(cp, dp + dm)[0, 1])},
           "profitable_cp": PROFITABLE, "n_pairs": len(pairs), "n_profitable": int((cp >= PROFITABLE).sum())}
    table, lost, best_cell = {}, {}, None
    for am in AM:
        for ap in AP:
            pruned = [p for p, a, b in zip(pairs, dp, dm) if a < ap and b < am]   # R9: AND, strict
            n_lost = sum(1 for p in pruned if best[p] >= PROFITABLE)
            table[f"{am}|{ap}"] = len(pruned)
            lost[f"{am}|{ap}"] = n_lost
            if n_lost == 0 and (best_cell is None or len(pruned) > best_cell[2]):
                best_cell = (ap, am, len(pruned))
    res["pruning_table"] = {"rows_alpha_m": AM, "cols_alpha_p": AP,
                            "pruned": [[table[f"{am}|{ap}"] for ap in AP] for am in AM],
                            "profitable_pruned": [[lost[f"{am}|{ap}"] for ap in AP] for am in AM]}
    res["paper_defaults"] = {"alpha_p": 0.4, "alpha_m": 0.1, "pruned": sum(1 for a, b in zip(dp, dm) if a < 0.4 and b < 0.1),
                             "profitable_pruned": sum(1 for p, a, b in zip(pairs, dp, dm)
                                                      if a < 0.4 and b < 0.1 and best[p] >= PROFITABLE)}
    if best_cell:
        res["b200_defaults"] = {"alpha_p": best_cell[0], "alpha_m": best_cell[1], "pruned": best_cell[2],
                                "rule": f"most pairs pruned with no pair of best measured CP >= {PROFITABLE} pruned"}
    res["p_percent_rule"] = {k: {"m_min": calib["profiles"][k].get("m_min"),
                                 "overhead_by_waves": calib["measured"].get(k, {}).get("slicing_overhead")}
                             for k in KINDS}
    print(json.dumps({k: res[k] for k in ("correlation", "paper_defaults", "b200_defaults", "n_profitable")}, indent=1))
    for am, row, lrow in zip(AM, res["pruning_table"]["pruned"], res["pruning_table"]["profitable_pruned"]):
        print(f"{am:6.3f} " + " ".join(f"{v:3d}/{l}" for v, l in zip(row, lrow)))
    json.dump(res, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01_pruning_b200.json"))

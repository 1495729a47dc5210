#!/usr/bin/env python
"""Per co-scheduled slice evidence from one timed bench step (north_star: achieved HBM GB/s,
issue/pipe rate and achieved occupancy per co-scheduled slice).  CPU post-processing of
`bench.py --trace-out` (device %globaltimer records of every launch: vb range, admission cap,
per-SM residency high-water mark from the %smid admission counters, partner).

ncu's kernel replay serialises concurrent kernels, so per-slice rates come from the device
records: a launch's algorithmic work (bench.algorithmic_work per virtual block x executed blocks)
over its resident interval.  The aggregate timeline sums every resident launch's rate per 10 us
bin: the HBM bandwidth and MUFU rate the co-schedule sustains as a whole.

usage: python tools/slice_report.py TRACE.jsonl [OUT.json] [--sm-mhz 1965]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import kl_inputs as G  # noqa: E402


def per_block_work(kind: str) -> dict:
    p = dict(G.PAPER[kind])
    w = bench.algorithmic_work(kind, p)
    g = G.grid_blocks(kind, p)
    return {k: (v / g if isinstance(v, (int, float)) else v) for k, v in w.items()}


def main(path: str, out: str | None, sm_mhz: float) -> dict:
    recs = [json.loads(line) for line in open(path) if line.strip()]
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = json.load(open(peaks_path)) if os.path.exists(peaks_path) else {"hbm_gbs": 6539.9, "bf16_tflops": 1671.8}
    rows = []
    for r in recs:
        if r["kind"] not in G.PAPER or r["t1_us"] <= r["t0_us"] or r["end"] <= r["start"]:
            continue
        w = per_block_work(r["kind"])
        blocks = r["end"] - r["start"]
        dt = (r["t1_us"] - r["t0_us"]) * 1e-6
        row = {"kind": r["kind"], "partner": r["partner"], "cap": r["cap"], "cap_max": r.get("cap_max", r["cap"]),
               "residency_max_per_sm": r.get("mx"),
               "blocks": blocks, "t0_us": r["t0_us"], "t1_us": r["t1_us"], "bound": w["bound"]}
        row["hbm_GBps"] = w.get("bytes", 0.0) * blocks / dt / 1e9
        if w["bound"] == "alu":
            pk, unit = bench.alu_peak(r["kind"], sm_mhz)
            row["alu_rate"] = w["ops"] * blocks / dt
            row["alu_frac"] = row["alu_rate"] / pk
            row["alu_unit"] = unit
        if w["bound"] == "tensor":
            row["tflops"] = w["flops"] * blocks / dt / 1e12
            row["tensor_frac"] = row["tflops"] / peaks["bf16_tflops"]
        row["hbm_frac"] = row["hbm_GBps"] / peaks["hbm_gbs"]
        rows.append(row)
    # aggregate timeline (10 us bins): sum of the resident launches' uniform rates
    t_end = max(r["t1_us"] for r in rows)
    nb = int(t_end // 10) + 1
    hbm = [0.0] * nb
    mufu = [0.0] * nb
    for r in rows:
        a, z = r["t0_us"], r["t1_us"]
        for b in range(int(a // 10), min(nb, int(z // 10) + 1)):
            ov = max(0.0, min(z, (b + 1) * 10) - max(a, b * 10)) / 10
            hbm[b] += r["hbm_GBps"] * ov
            if r["kind"] == "MRIQ":
                mufu[b] += r["alu_frac"] * ov
    co = [r for r in rows if r["partner"]]
    occ = [r for r in co if r["cap_max"] and r["residency_max_per_sm"] is not None]
    res = {
        "source": os.path.basename(path),
        "how": __doc__.split("\n\n")[1].replace("\n", " "),
        "peaks": {"hbm_GBps": peaks["hbm_gbs"], "bf16_tflops": peaks["bf16_tflops"], "sm_mhz": sm_mhz},
        "launches": len(rows), "co_scheduled_launches": len(co),
        "residency_reaches_cap": sum(1 for r in occ if r["residency_max_per_sm"] == r["cap_max"]),
        "residency_above_cap": sum(1 for r in occ if r["residency_max_per_sm"] > r["cap_max"]),
        "residency_checked": len(occ),
        "aggregate": {"step_us": t_end, "mean_hbm_GBps": sum(hbm) / nb, "mean_hbm_frac": sum(hbm) / nb / peaks["hbm_gbs"],
                      "peak_bin_hbm_GBps": max(hbm), "mean_mriq_mufu_frac": sum(mufu) / nb},
        "slices": rows,
    }
    if out:
        with open(out, "w") as f:
            json.dump(res, f, indent=1)
    return res


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    mhz = float(sys.argv[sys.argv.index("--sm-mhz") + 1]) if "--sm-mhz" in sys.argv else 1965.0
    if "--sm-mhz" in sys.argv:
        args = [a for a in args if a != str(sys.argv[sys.argv.index("--sm-mhz") + 1])]
    r = main(args[0], args[1] if len(args) > 1 else None, mhz)
    print(json.dumps({k: v for k, v in r.items() if k not in ("slices", "how")}, indent=1))
    for s in r["slices"]:
        extra = f"alu {s['alu_frac']:.2f}" if "alu_frac" in s else (f"tensor {s['tensor_frac']:.2f}" if "tensor_frac" in s else "")
        print(f"{s['kind']:5s} with {str(s['partner']):5s} cap {s['cap']:2d} resid {s['residency_max_per_sm']} "
              f"{s['t0_us']:8.1f}-{s['t1_us']:8.1f} us blocks {s['blocks']:6d} HBM {s['hbm_GBps']:7.0f} GB/s {extra}")

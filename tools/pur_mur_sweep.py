#!/usr/bin/env python
"""f4 synthetic PUR/MUR study (Fig. pur_mur): "testing kernels" mixing memory and
computation -- the synthetic streaming kernel (one float4 load + c dependent FMAs per component +
one store) at c in FMAS -- measured solo for PUR (warp instructions issued per cycle per virtual
SM, ncu smsp__inst_executed over the kernel's cycles) and MUR (DRAM bytes over time at the measured
HBM peak), then co-run pairwise through the slice launcher (kl_run_pair, 4 + 4 blocks per SM) for
the measured CP (Eq.1 from each kernel's progress rate relative to solo).  Reports CP against
|dPUR| and |dMUR|.
usage: python tools/pur_mur_sweep.py [out.json]     (needs a GPU and ncu)"""
import csv
import io
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

FMAS = [0, 2, 8, 24, 64, 160]
N = 1 << 26


def ncu_solo(fmas):
    """PUR and MUR of one solo plain launch, from ncu (cold L2, counters)."""
    code = ("import sys,os;sys.path.insert(0,os.getcwd());import torch,kl_inputs as G,paper_1303_5164_b200 as K;"
            "from paper_1303_5164_b200.workload import Instance;ctx=K.Context(device=0);"
            f"i=Instance(G.gen('SYNTH',dict(n={N},fmas={fmas})),'cuda');"
            "ctx.run_plain('SYNTH',i.grid,i.args,0);ctx.run_plain('SYNTH',i.grid,i.args,0);torch.cuda.synchronize()")
    out = subprocess.run(["ncu", "--metrics", "smsp__inst_executed.sum,sm__cycles_elapsed.avg,dram__bytes_read.sum,"
                          "dram__bytes_write.sum,gpu__time_duration.sum", "-k", "regex:k_plain", "-s", "1", "-c", "1", "--csv",
                          sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT).stdout
    rows = list(csv.reader(io.StringIO("\n".join(l for l in out.splitlines() if l.startswith('"')))))
    h = rows[0]
    m = {}
    for r in rows[1:]:
        v = float(r[h.index("Metric Value")].replace(",", ""))
        unit = r[h.index("Metric Unit")]
        mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
               "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
               "second": 1.0, "s": 1.0}.get(unit, 1.0)
        m[r[h.index("Metric Name")]] = v * mul
    return m


def main(out_path):
    import torch

    import kl_inputs as G
    import paper_1303_5164_b200 as K
    from paper_1303_5164_b200.workload import Instance
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6540.0}
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    solo = {}
    for c in FMAS:
        m = ncu_solo(c)
        pur = m["smsp__inst_executed.sum"] / (m["sm__cycles_elapsed.avg"] * 4 * n_sm)
        mur = (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / m["gpu__time_duration.sum"] / (peaks["hbm_gbs"] * 1e9)
        solo[c] = {"pur": pur, "mur": mur, "ncu": m}
        print("fmas", c, "PUR", round(pur, 3), "MUR", round(mur, 3), flush=True)
    ctx = K.Context(device=0)
    insts = {c: Instance(G.gen("SYNTH", dict(n=N, fmas=c)), "cuda") for c in FMAS}
    rate = {}
    for c in FMAS:                       # solo progress rate at full occupancy (blocks / ns)
        i = insts[c]
        ctx.run_capped("SYNTH", i.grid, i.args, 0)
        ms = ctx.run_capped("SYNTH", i.grid, i.args, 0)
        rate[c] = i.grid / (ms * 1e6)
    pairs = []
    for a, b in itertools.combinations(FMAS, 2):
        ia, ib = insts[a], insts[b]
        ra, rb = ctx.run_pair("SYNTH", ia.grid, ia.args, 4, "SYNTH", ib.grid, ib.args, 4)
        pa = ra.executed / max(ra.t1_ns - ra.t0_ns, 1) / rate[a]
        pb = rb.executed / max(rb.t1_ns - rb.t0_ns, 1) / rate[b]
        cp = 1.0 - 1.0 / (pa + pb)
        pairs.append({"a": a, "b": b, "cp": cp, "dpur": abs(solo[a]["pur"] - solo[b]["pur"]),
                      "dmur": abs(solo[a]["mur"] - solo[b]["mur"])})
        print(a, b, "CP", round(cp, 3), "dPUR", round(pairs[-1]["dpur"], 3), "dMUR", round(pairs[-1]["dmur"], 3),
              flush=True)
    cp = np.array([p["cp"] for p in pairs])
    dp = np.array([p["dpur"] for p in pairs])
    dm = np.array([p["dmur"] for p in pairs])
    res = {"fmas": FMAS, "n": N, "solo": {str(k): v for k, v in solo.items()},
           "pairs": pairs, "pearson_cp_dpur": float(np.corrcoef(cp, dp)[0, 1]),
           "pearson_cp_dmur": float(np.corrcoef(cp, dm)[0, 1]), "how": __doc__.split("\n")[0]}
    print(json.dumps({k: res[k] for k in ("pearson_cp_dpur", "pearson_cp_dmur")}))
    json.dump(res, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "pur_mur_sweep.json"))

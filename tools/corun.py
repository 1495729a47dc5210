"""Co-run measurement shared by the OPT table (f2) and the model-error study (C3): both kernels run
concurrently through the slice launcher (kl_run_pair, each at its cap), every block's start and end
are recorded on the device (config.audit = 2, kl_timeline), and each kernel's progress is counted
inside the window where both are resident -- from the later first-block start to the earlier
last-block end -- with blocks that straddle a window edge credited by the fraction of their
duration inside it; when that window covers less than half of the shorter run (a short kernel
ending while its partner ramps up), each kernel's own run is used.  Progress rates are blocks per ns; the solo rate of a kind is measured the
same way at its solo occupancy."""
import numpy as np


def progress(tl, t0, t1):
    """Blocks of timeline tl (grid x 2: start, end) completed inside [t0, t1], edge blocks pro rata."""
    s, e = tl[:, 0].astype(np.float64), tl[:, 1].astype(np.float64)
    ran = e > 0
    s, e = s[ran], e[ran]
    ov = np.clip(np.minimum(e, t1) - np.maximum(s, t0), 0.0, None)
    dur = np.maximum(e - s, 1.0)
    return float((ov / dur).sum())


def span(tl):
    ran = tl[:, 1] > 0
    return int(tl[ran, 0].min()), int(tl[ran, 1].max())


def solo_rate(ctx, kind, inst, cap):
    """Blocks per ns of `kind` alone at `cap` blocks per SM, from its own block timestamps (first
    block start to last block end; no launch latency), second of two runs."""
    rate = 0.0
    for _ in range(2):
        ctx.run_capped(kind, inst.grid, inst.args, cap)
        tl = ctx.timeline(ctx.trace()[-1].id, inst.grid)
        a, z = span(tl)
        rate = inst.grid / max(z - a, 1)
    return rate


def corun(ctx, k1, i1, b1, k2, i2, b2, min_overlap=0.5):
    """Co-run k1 (cap b1) with k2 (cap b2); returns (rate1, rate2, window_ns) in blocks/ns.
    When the common window covers less than `min_overlap` of the shorter run (a short kernel that
    ends while its partner still ramps up), each kernel's own run is used instead."""
    r1, r2 = ctx.run_pair(k1, i1.grid, i1.args, b1, k2, i2.grid, i2.args, b2)
    tl1, tl2 = ctx.timeline(r1.id, i1.grid), ctx.timeline(r2.id, i2.grid)
    a1, z1 = span(tl1)
    a2, z2 = span(tl2)
    t0, t1 = max(a1, a2), min(z1, z2)
    if t1 - t0 >= min_overlap * min(z1 - a1, z2 - a2) and t1 > t0:
        w = float(t1 - t0)
        return progress(tl1, t0, t1) / w, progress(tl2, t0, t1) / w, int(w)
    n1, n2 = float((tl1[:, 1] > 0).sum()), float((tl2[:, 1] > 0).sum())
    return n1 / max(z1 - a1, 1), n2 / max(z2 - a2, 1), 0


# ---- steady-state co-runs -----------------------------------------------------------------
# At paper size the kinds' solo times span 21 us (SPMV) to 2 ms (MRIQ): a co-run of a short and a
# long kernel ends while the long one still ramps, and the window rates are dominated by ramp and
# tail blocks (round-2 tables had rates of 1 % of solo for MRIQ beside SAD).  The steady mode runs
# every kind at a size scaled along its independent dimension so its solo run takes >= target.
SCALE_DIM = {"PC": "n_threads", "SAD": "height", "SPMV": "n_rows", "ST": "nz", "MM": "M", "MRIQ": "num_x",
             "BS": "n", "TEA": "n", "SYNTH": "n", "MATADD": None}


def scaled_size(kind, s):
    import kl_inputs as G
    p = dict(G.PAPER[kind])
    dim = SCALE_DIM.get(kind)
    if dim and s > 1:
        p[dim] = p[dim] * s
    return p


def steady_instances(kinds, solo_ms, target_ms=2.0, device="cuda"):
    """One instance per kind sized so that its solo run takes about target_ms (solo_ms: paper-size
    solo time per kind)."""
    import math
    import kl_inputs as G
    from paper_1303_5164_b200.workload import Instance
    out = {}
    for k in kinds:
        s = max(1, int(math.ceil(target_ms / max(solo_ms[k], 1e-3))))
        out[k] = Instance(G.gen(k, scaled_size(k, s)), device)
        out[k].scale = s
    return out

"""Host-side logic of the measurement tools (CPU): co-run window accounting (tools/corun.py)."""
import numpy as np

from tools.corun import progress, span


def test_progress_full_and_partial_blocks():
    # three blocks: fully inside, straddling the window end (half inside), outside; one never ran
    tl = np.array([[100, 200], [250, 350], [400, 500], [0, 0]], dtype=np.int64)
    assert span(tl) == (100, 500)
    assert abs(progress(tl, 100, 300) - 1.5) < 1e-12
    assert abs(progress(tl, 0, 1000) - 3.0) < 1e-12
    assert progress(tl, 600, 700) == 0.0


def test_progress_rate_of_uniform_stream():
    # a kernel completing one block every 10 ns for 1000 blocks: 0.1 blocks/ns in any window
    s = np.arange(1000, dtype=np.int64) * 10 + 5
    tl = np.stack([s, s + 10], axis=1)
    for t0, t1 in ((1000, 3000), (1234, 8765)):
        assert abs(progress(tl, t0, t1) / (t1 - t0) - 0.1) < 1e-9


def test_slice_report_rates_and_residency(tmp_path):
    """tools/slice_report.py: per-slice algorithmic rate = work per virtual block x executed
    blocks / resident interval; residency checked against the admission cap; aggregate HBM
    timeline sums concurrent slices."""
    import json
    import kl_inputs as G
    from tools import slice_report as SR
    p = dict(G.PAPER["PC"])
    g = G.grid_blocks("PC", p)
    recs = [{"kind": "PC", "cap": 4, "cap_max": 4, "start": 0, "end": g, "exh": 1, "adm": 592, "mx": 4,
             "t0_us": 0.0, "t1_us": 500.0, "partner": "MRIQ", "cp": 0.2, "dec": 1},
            {"kind": "MRIQ", "cap": 4, "cap_max": 4, "start": 0, "end": 100, "exh": 0, "adm": 592, "mx": 5,
             "t0_us": 0.0, "t1_us": 500.0, "partner": "PC", "cp": 0.2, "dec": 1}]
    f = tmp_path / "t.jsonl"
    f.write_text("\n".join(json.dumps(r) for r in recs) + "\n")
    r = SR.main(str(f), None, 1965.0)
    pc = next(s for s in r["slices"] if s["kind"] == "PC")
    want = p["n_threads"] * (p["hops"] * 64 + 8) / 500e-6 / 1e9      # whole PC in 500 us
    assert abs(pc["hbm_GBps"] - want) < 1e-6 * want
    assert r["residency_checked"] == 2 and r["residency_reaches_cap"] == 1 and r["residency_above_cap"] == 1
    assert r["aggregate"]["peak_bin_hbm_GBps"] >= pc["hbm_GBps"]


def test_johnson_order_minimises_two_stage_makespan():
    """bench.johnson_order (e2e copy order): on random two-machine flow shops its makespan equals
    the brute-force minimum over all job orders (Johnson 1954)."""
    import itertools
    import random
    import bench

    def makespan(order, a, b):
        t1 = t2 = 0.0
        for j in order:
            t1 += a[j]
            t2 = max(t2, t1) + b[j]
        return t2

    rng = random.Random(7)
    for _ in range(200):
        jobs = list(range(6))
        a = {j: rng.uniform(0.1, 10) for j in jobs}
        b = {j: rng.uniform(0.1, 10) for j in jobs}
        best = min(makespan(p, a, b) for p in itertools.permutations(jobs))
        assert abs(makespan(bench.johnson_order(jobs, a, b), a, b) - best) < 1e-9

"""Pins of the oracle's benchmark kernels (oracle/kernels.c): closed forms, invariants, exact
integer cases and published vectors -- each chosen so that a dropped term, a wrong sign or index,
or a transposed operand fails one of them."""
import math

import numpy as np
import pytest

import kl_inputs as G
import oracle as O


def test_pc_closed_form_cycle():
    """next[i] = i+1 mod N: after H hops out = (start + H) mod N, acc = sum_{j=1..H}(start+j mod N)."""
    d = G.gen("PC", "small", mode="cycle")
    p = d["params"]
    r = O.run_kernel(d)
    t = np.arange(p["n_threads"], dtype=np.uint64)
    start = ((t * np.uint64(2654435761)) & np.uint64(0xFFFFFFFF)) % np.uint64(p["n_nodes"])
    H = p["hops"]
    assert np.array_equal(r["out"].astype(np.uint64), (start + np.uint64(H)) % np.uint64(p["n_nodes"]))
    acc = np.zeros_like(start)
    for j in range(1, H + 1):
        acc = (acc + (start + np.uint64(j)) % np.uint64(p["n_nodes"])) & np.uint64(0xFFFFFFFF)
    assert np.array_equal(r["acc"].astype(np.uint64), acc)


def test_pc_random_cycle_and_sample():
    d = G.gen("PC", "small")
    nxt = d["next"].astype(np.int64)
    # generator invariant: one cycle through all N nodes
    seen, p = 0, 0
    for _ in range(nxt.size):
        p = nxt[p]
        seen += 1
        if p == 0:
            break
    assert seen == nxt.size
    full = O.run_kernel(d)
    idx = np.array([0, 5, 777, d["params"]["n_threads"] - 1])
    s = O.run_kernel(d, idx)
    assert np.array_equal(s["out"], full["out"][idx]) and np.array_equal(s["acc"], full["acc"][idx])


def test_sad_identical_and_shift():
    """Identical frames: SAD = 0 at zero displacement (16,16).  ref(x+u, y+v) = cur(x, y):
    SAD = 0 at (16+u, 16+v) for macroblocks whose window needs no clamping."""
    d = G.gen("SAD", "small", mode="identical")
    r = O.run_kernel(d)["sad"].reshape(-1, 33, 33)
    assert np.all(r[:, 16, 16] == 0)
    assert r.max() <= 255 * 256
    u, v = 3, -5
    d = G.gen("SAD", "small", mode="shift", u=u, v=v)
    r = O.run_kernel(d)["sad"].reshape(-1, 33, 33)
    mbw, mbh = 176 // 16, 112 // 16
    for my in range(1, mbh - 1):
        for mx in range(1, mbw - 1):
            m = my * mbw + mx
            assert r[m, 16 + v, 16 + u] == 0
            assert r[m, 16, 16] > 0


def test_sad_edge_clamp_numpy():
    """Independent formulation: numpy edge padding (= clamped reference) on a tiny frame."""
    d = G.gen("SAD", {"width": 48, "height": 32}, seed=3)
    r = O.run_kernel(d)["sad"].reshape(-1, 33, 33)
    cur, ref = d["cur"].astype(np.int64), d["ref"].astype(np.int64)
    pad = np.pad(ref, 16, mode="edge")
    for m in range(r.shape[0]):
        mx, my = m % 3, m // 3
        blk = cur[my * 16:(my + 1) * 16, mx * 16:(mx + 1) * 16]
        for dy in (0, 7, 16, 32):
            for dx in (0, 11, 16, 32):
                win = pad[my * 16 + dy:my * 16 + dy + 16, mx * 16 + dx:mx * 16 + dx + 16]
                assert r[m, dy, dx] == np.abs(blk - win).sum()


def test_spmv_identity_and_integer():
    d = G.gen("SPMV", {"n_rows": 500, "n_cols": 600, "nnz_min": 8, "nnz_max": 24}, mode="identity")
    assert np.array_equal(O.run_kernel(d)["y"], d["x"][:500])
    d = G.gen("SPMV", "small", mode="int")
    y = O.run_kernel(d)["y"]
    rp, c, v, x = d["rowptr"], d["cols"], d["vals"].astype(np.int64), d["x"].astype(np.int64)
    prod = v * x[c]
    ref = np.add.reduceat(prod, rp[:-1]) if prod.size else np.zeros(0)
    ref[np.diff(rp) == 0] = 0
    assert np.array_equal(y.astype(np.int64), ref)


def test_stencil_laplacian_modes():
    """c1 = 1, c0 = 6 turns the 7-point stencil into the discrete Laplacian: exactly 0 on a
    linear field in the interior, integer-exact on integer fields; boundary copies the input."""
    d = G.gen("ST", "small", mode="linear")
    nx, ny, nz = (d["params"][k] for k in ("nx", "ny", "nz"))
    out = O.run_kernel(d, c0=6.0, c1=1.0)["out"].reshape(nz, ny, nx)
    a = d["inp"]
    assert np.all(out[1:-1, 1:-1, 1:-1] == 0)
    for sl in [(0,), (-1,), (slice(None), 0), (slice(None), -1), (Ellipsis, 0), (Ellipsis, -1)]:
        assert np.array_equal(out[sl], a[sl])
    d = G.gen("ST", "small", mode="int")
    out = O.run_kernel(d, c0=6.0, c1=1.0)["out"].reshape(nz, ny, nx).astype(np.int64)
    a = d["inp"].astype(np.int64)
    lap = (a[:-2, 1:-1, 1:-1] + a[2:, 1:-1, 1:-1] + a[1:-1, :-2, 1:-1] + a[1:-1, 2:, 1:-1]
           + a[1:-1, 1:-1, :-2] + a[1:-1, 1:-1, 2:] - 6 * a[1:-1, 1:-1, 1:-1])
    assert np.array_equal(out[1:-1, 1:-1, 1:-1], lap)


def test_stencil_parboil_constant_field():
    """Parboil constants c0 = 1/6, c1 = 1/36 on a constant field: 6 c1 - c0 = 0 up to fp32
    rounding of the constants."""
    d = G.gen("ST", {"nx": 8, "ny": 8, "nz": 8})
    d["inp"] = np.full((8, 8, 8), 3.0, np.float32)
    out = O.run_kernel(d)["out"].reshape(8, 8, 8)
    assert np.max(np.abs(out[1:-1, 1:-1, 1:-1])) < 1e-6


def test_mm_integer_exact():
    d = G.gen("MM", "small", mode="int")
    C = O.run_kernel(d)["C"].reshape(512, 256)
    A = (d["A"].astype(np.uint32) << 16).view(np.float32).astype(np.int64)
    Bt = (d["Bt"].astype(np.uint32) << 16).view(np.float32).astype(np.int64)
    assert np.array_equal(C.astype(np.int64), A @ Bt.T)


def test_mriq_special_cases():
    d = G.gen("MRIQ", "small", mode="zero_k")
    r = O.run_kernel(d)
    s = float(np.sum(d["phimag"].astype(np.float64)))
    assert np.allclose(r["qr"], s, rtol=1e-6) and np.all(np.abs(r["qi"]) < 1e-6)
    # one k-point (1,0,0) and x = 0.25: phase 2 pi * 0.25 -> Qr = 0, Qi = phiMag
    d = G.gen("MRIQ", {"num_x": 4, "num_k": 1})
    d["x"] = np.full(4, 0.25, np.float32); d["y"] = np.zeros(4, np.float32); d["z"] = np.zeros(4, np.float32)
    d["kx"] = np.ones(1, np.float32); d["ky"] = np.zeros(1, np.float32); d["kz"] = np.zeros(1, np.float32)
    d["phimag"] = np.full(1, 1.5, np.float32)
    r = O.run_kernel(d)
    assert np.all(np.abs(r["qr"]) < 1e-7) and np.allclose(r["qi"], 1.5)
    # y and z enter: k = (0, 2, 0), y = 0.5 -> integer phase, cos = 1
    d["x"][:] = 0.0; d["y"][:] = 0.5; d["kx"][:] = 0.0; d["ky"][:] = 2.0
    r = O.run_kernel(d)
    assert np.allclose(r["qr"], 1.5) and np.all(np.abs(r["qi"]) < 1e-6)


def test_bs_cnd_and_parity():
    """A&S 26.2.17 is within 7.5e-8 of the normal CDF (0.5 erfc(-d/sqrt 2)); CND(d)+CND(-d)=1;
    put-call parity C - P = S - X e^{-RT}."""
    for dd in np.linspace(-8, 8, 161):
        ref = 0.5 * math.erfc(-dd / math.sqrt(2))
        assert abs(O.cnd(dd) - ref) < 7.5e-8
        if dd != 0:   # at d = 0 both sides are the same tail value (~0.5 - 5e-10)
            assert abs(O.cnd(dd) + O.cnd(-dd) - 1) < 1e-15
    d = G.gen("BS", "small")
    r = O.run_kernel(d)
    S, X, T = (d[k].astype(np.float64) for k in "SXT")
    parity = S - X * np.exp(-0.02 * T)
    assert np.max(np.abs(r["call"] - r["put"] - parity) / r["scale"]) < 1e-6
    assert np.all(r["call"] >= -1e-6) and np.all(r["put"] >= -1e-6)
    # deep in the money, T small: call ~ S - X e^{-RT}
    d2 = G.gen("BS", {"n": 4})
    d2["S"] = np.full(4, 30.0, np.float32); d2["X"] = np.full(4, 1.0, np.float32); d2["T"] = np.full(4, 0.25, np.float32)
    r2 = O.run_kernel(d2)
    assert np.allclose(r2["call"], 30.0 - math.exp(-0.02 * 0.25), rtol=1e-6)


def test_bs_textbook_value():
    """Pins d1 = (ln(S/X) + (R + V^2/2) T) / (V sqrt T) and d2 = d1 - V sqrt T through a printed
    textbook example (tests/golden/bs_textbook.txt): put-call parity holds for any d1/d2 and the
    deep-in-the-money case saturates CND, so only printed prices catch a wrong drift or V sqrt T.
    The A&S CND error (< 7.5e-8) is far below the printed rounding (0.005)."""
    f = open(__file__.replace("test_oracle_kernels.py", "golden/bs_textbook.txt")).read().split("\n")
    rows = [list(map(float, l.split())) for l in f if l.strip() and not l.startswith("#")]
    for S, X, R, V, T, d1, d2, call, put in rows:
        d = G.gen("BS", {"n": 2})
        d["S"] = np.full(2, S, np.float32); d["X"] = np.full(2, X, np.float32); d["T"] = np.full(2, T, np.float32)
        d["params"].update(R=R, V=V)
        r = O.run_kernel(d)
        assert np.all(np.abs(r["call"] - call) < 0.005), (r["call"], call)
        assert np.all(np.abs(r["put"] - put) < 0.005), (r["put"], put)
        # d1 and d2 separately: N(d1) = dC/dS and N(d2) = -e^{RT} dC/dX, by central differences
        # of the oracle's own prices (fp32 inputs: steps large enough to be exactly representable)
        h = 0.25
        dd = G.gen("BS", {"n": 4})
        dd["S"] = np.array([S + h, S - h, S, S], np.float32); dd["X"] = np.array([X, X, X + h, X - h], np.float32)
        dd["T"] = np.full(4, T, np.float32); dd["params"].update(R=R, V=V)
        c = O.run_kernel(dd)["call"].astype(np.float64)
        n_d1 = (c[0] - c[1]) / (2 * h)
        n_d2 = -(c[2] - c[3]) / (2 * h) * math.exp(R * T)
        assert abs(n_d1 - 0.5 * math.erfc(-d1 / math.sqrt(2))) < 2e-3, n_d1
        assert abs(n_d2 - 0.5 * math.erfc(-d2 / math.sqrt(2))) < 2e-3, n_d2


def test_tea_known_answer_and_roundtrip():
    f = open(__file__.replace("test_oracle_kernels.py", "golden/tea_kat.txt")).read().split("\n")
    line = [l for l in f if l and not l.startswith("#")][0].split()
    vals = [int(x, 16) for x in line]
    d = G.gen("TEA", {"n": 1})
    d["key"] = np.array(vals[0:4], np.uint32)
    d["v"] = np.array(vals[4:6], np.uint32)
    assert list(O.run_kernel(d)["out"]) == vals[6:8]
    d = G.gen("TEA", "small")
    enc = O.run_kernel(d)["out"]
    assert np.array_equal(O.tea_decrypt(enc, d["key"]), d["v"])
    assert not np.array_equal(enc, d["v"])


def test_matadd_and_synth():
    d = G.gen("MATADD", "small")
    assert np.array_equal(O.run_kernel(d)["C"], d["A"] + d["B"])
    d = G.gen("SYNTH", "small")
    d["params"].update(a=0.5, b=0.0, fmas=3)
    assert np.array_equal(O.run_kernel(d)["y"], d["x"] / 8)
    d["params"].update(fmas=0)
    assert np.array_equal(O.run_kernel(d)["y"], d["x"])

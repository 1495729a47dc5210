"""Pins of the f1 three-state (coalesced / uncoalesced) model oracle (oracle/model3.c,
PAPER.md P:1000-1019, reading R27 in DESIGN.md §3), against things other than the oracle itself:

* reductions the paper's wording implies: with no uncoalesced accesses (uc = 0), or with both
  access classes alike (ru = r, equal latencies), the chain is exactly the two-state chain
  (the three-state model "extends" the two-state one) -- solo and joint;
* a closed form: one warp (W = 1), state-dependent latencies: IPC = 1/(1 + Rm(1-uc)/P_c + Rm uc/P_u);
* invariants: row-stochastic, pi P = pi, symmetry of the joint chain, lumpability of two identical
  kernels into one kernel with w1 + w2 warps;
* an independent per-warp Monte Carlo simulation of the three-state round process (each ready
  warp issues and stalls coalesced / uncoalesced / not, each idle warp returns with its class's
  probability), within 3.5 sigma of batch means.
"""
import math

import numpy as np
import pytest

import oracle as O


def _cfg(**kw):
    base = dict(L0=300.0, B=1.0, a0=1.0, b0=0.0, W=16)
    base.update(kw)
    return O.SmCfg(base["L0"], base["B"], base["a0"], base["b0"], base["W"], 0, 0, 0.0)


@pytest.mark.parametrize("w,c,u", [(6, 0, 0), (6, 2, 3), (8, 8, 0), (5, 0, 5), (16, 4, 7)])
def test_rows_stochastic(w, c, u):
    k = O.kmodel3(0.2, r=2.0, uc=0.4, ru=12.0)
    r = O.row3(k, w, c, u, 0.3, 0.05)
    assert abs(r.sum() - 1.0) < 1e-12 and r.min() >= 0.0
    # states with more idle warps than the kernel has are never produced
    assert len(r) == O.nstates3(w) == (w + 1) * (w + 2) // 2


def test_stationary_is_left_eigenvector():
    cfg = _cfg()
    P, R = O.build3(O.kmodel3(0.15, r=2.0, uc=0.3, ru=16.0), 5, cfg, O.kmodel3(0.05, r=1.0, uc=0.1, ru=8.0), 4)
    assert np.abs(P.sum(1) - 1.0).max() < 1e-12
    pi = O.stationary(P)
    assert abs(pi.sum() - 1.0) < 1e-12 and pi.min() > -1e-15
    assert np.abs(pi @ P - pi).max() < 1e-12


@pytest.mark.parametrize("w,rm,r", [(1, 0.5, 1.0), (6, 0.1, 2.0), (16, 0.02, 4.0), (9, 0.3, 8.0)])
def test_uc_zero_is_two_state(w, rm, r):
    cfg = _cfg()
    P2, R2 = O.build_homog(O.kmodel(rm, r=r), w, cfg)
    two = O.ipc_homog(w, O.stationary(P2), R2)
    P3, R3 = O.build3(O.kmodel3(rm, r=r, uc=0.0, ru=32.0), w, cfg)
    assert abs(O.ipc3(w, O.stationary(P3), R3) - two) < 1e-12


@pytest.mark.parametrize("uc", [0.0, 0.25, 1.0])
def test_equal_classes_are_two_state(uc):
    """ru = r: both idle classes return alike, so (c, u) lumps to c + u = two-state idle count."""
    cfg = _cfg(L0=200.0, a0=2.0)
    w = 8
    P2, R2 = O.build_homog(O.kmodel(0.12, r=3.0), w, cfg)
    two = O.ipc_homog(w, O.stationary(P2), R2)
    P3, R3 = O.build3(O.kmodel3(0.12, r=3.0, uc=uc, ru=3.0), w, cfg)
    pi3 = O.stationary(P3)
    assert abs(O.ipc3(w, pi3, R3) - two) < 1e-12
    # and the lumped distribution is the two-state one
    lumped = np.zeros(w + 1)
    for s, (c, u) in enumerate(O.states3(w)):
        lumped[c + u] += pi3[s]
    assert np.abs(lumped - O.stationary(P2)).max() < 1e-12


def test_joint_uc_zero_is_two_state():
    cfg = _cfg(L0=150.0, a0=1.5)
    k1, k2 = O.kmodel(0.25, r=2.0), O.kmodel(0.05, r=1.0)
    P, R = O.build_joint(k1, 6, k2, 10, cfg)
    a, b, _ = O.ipc_joint(6, 10, O.stationary(P), R)
    P3, R3 = O.build3(O.kmodel3(0.25, r=2.0, uc=0.0, ru=20.0), 6, cfg, O.kmodel3(0.05, r=1.0, uc=0.0, ru=9.0), 10)
    a3, b3 = O.ipc3(6, O.stationary(P3), R3, w2=10)
    assert abs(a3 - a) < 1e-12 and abs(b3 - b) < 1e-12


@pytest.mark.parametrize("rm,uc,r,ru", [(0.5, 0.5, 1.0, 8.0), (0.2, 1.0, 2.0, 32.0), (0.9, 0.1, 1.0, 4.0)])
def test_w1_closed_form(rm, uc, r, ru):
    """One warp: R = 1 in every state; pi_C = pi_R Rm(1-uc)/P_c, pi_U = pi_R Rm uc/P_u, with the
    return probabilities evaluated in the idle state itself (n = r resp. ru outstanding)."""
    L0, a0, B = 20.0, 1.0, 0.5
    cfg = _cfg(L0=L0, a0=a0, B=B, W=1)
    Lc = L0 + a0 * r / B
    Lu = L0 + a0 * ru / B + a0 * (ru - r) / B
    expect = 1.0 / (1.0 + rm * (1 - uc) * Lc + rm * uc * Lu)
    P, R = O.build3(O.kmodel3(rm, r=r, uc=uc, ru=ru), 1, cfg)
    assert abs(O.ipc3(1, O.stationary(P), R) - expect) < 1e-13


def test_joint_symmetry():
    cfg = _cfg(L0=250.0, a0=1.0)
    ka, kb = O.kmodel3(0.2, r=2.0, uc=0.5, ru=16.0), O.kmodel3(0.05, r=1.0, uc=0.0, ru=1.0)
    P, R = O.build3(ka, 4, cfg, kb, 6)
    a, b = O.ipc3(4, O.stationary(P), R, w2=6)
    P, R = O.build3(kb, 6, cfg, ka, 4)
    b2, a2 = O.ipc3(6, O.stationary(P), R, w2=4)
    assert abs(a - a2) < 1e-12 and abs(b - b2) < 1e-12


@pytest.mark.parametrize("w1,w2", [(2, 3), (4, 4), (1, 6)])
def test_lumpability_identical_kernels(w1, w2):
    """Two instances of one kind split (w1, w2) behave as one kind with w1 + w2 warps (the
    latency depends on the total outstanding requests, the round on the total ready warps)."""
    cfg = _cfg(L0=180.0, a0=1.0)
    k = O.kmodel3(0.15, r=2.0, uc=0.3, ru=10.0)
    P, R = O.build3(k, w1, cfg, k, w2)
    a, b = O.ipc3(w1, O.stationary(P), R, w2=w2)
    Ph, Rh = O.build3(k, w1 + w2, cfg)
    assert abs((a + b) - O.ipc3(w1 + w2, O.stationary(Ph), Rh)) < 1e-11
    assert abs(a / w1 - b / w2) < 1e-11


def _simulate3(ws, kinds, L0, a0, B, rounds, seed):
    """Per-warp Monte Carlo of the three-state round process (independent of the chain code):
    warp state 0 ready, 1 coalesced-idle, 2 uncoalesced-idle."""
    rng = np.random.default_rng(seed)
    st = [np.zeros(w, np.int8) for w in ws]
    nb = 50
    per = rounds // nb
    inst_b, cyc_b = np.zeros(nb), np.zeros(nb)
    for bi in range(nb):
        inst = cyc = 0.0
        for _ in range(per):
            ready = sum(int((s == 0).sum()) for s in st)
            R = max(ready, 1)
            n = sum(float((s == 1).sum()) * k["r"] + float((s == 2).sum()) * k["ru"] for s, k in zip(st, kinds))
            Lc = L0 + a0 * n / B
            for i, (s, k) in enumerate(zip(st, kinds)):
                Lu = Lc + a0 * (k["ru"] - k["r"]) / B
                pc, pu = min(1.0, R / Lc), min(1.0, R / Lu)
                x = rng.random(len(s))
                new = s.copy()
                rd = s == 0
                inst += float(rd.sum())
                new[rd & (x < k["rm"] * (1 - k["uc"]))] = 1
                new[rd & (x >= k["rm"] * (1 - k["uc"])) & (x < k["rm"])] = 2
                new[(s == 1) & (x < pc)] = 0
                new[(s == 2) & (x < pu)] = 0
                st[i] = new
            cyc += R
        inst_b[bi], cyc_b[bi] = inst, cyc
    ipc = inst_b.sum() / cyc_b.sum()
    return ipc, np.std(inst_b / cyc_b, ddof=1) / math.sqrt(nb)


def test_monte_carlo_solo():
    k = dict(rm=0.2, r=2.0, uc=0.4, ru=24.0)
    cfg = _cfg(L0=60.0, a0=1.0, B=2.0)
    P, R = O.build3(O.kmodel3(k["rm"], r=k["r"], uc=k["uc"], ru=k["ru"]), 6, cfg)
    model = O.ipc3(6, O.stationary(P), R)
    mc, sig = _simulate3([6], [k], 60.0, 1.0, 2.0, 60000, seed=3)
    assert abs(mc - model) <= 3.5 * sig + 1e-4, (mc, model, sig)


def test_monte_carlo_joint():
    k1 = dict(rm=0.25, r=2.0, uc=0.5, ru=16.0)
    k2 = dict(rm=0.05, r=1.0, uc=0.0, ru=1.0)
    cfg = _cfg(L0=80.0, a0=1.0, B=1.0)
    P, R = O.build3(O.kmodel3(**{a: k1[a] for a in k1}), 4, cfg, O.kmodel3(**{a: k2[a] for a in k2}), 4)
    a, b = O.ipc3(4, O.stationary(P), R, w2=4)
    mc, sig = _simulate3([4, 4], [k1, k2], 80.0, 1.0, 1.0, 60000, seed=5)
    assert abs(mc - (a + b)) <= 3.5 * sig + 1e-4, (mc, a + b, sig)


def test_uncoalesced_lowers_ipc():
    """The paper's observation: treating uncoalesced accesses as coalesced
    over-predicts IPC."""
    cfg = _cfg()
    two = O.solo_ipc3(O.kmodel3(0.1, r=2.0, uc=0.0, ru=32.0, wpb=8), 4, 4, cfg)
    three = O.solo_ipc3(O.kmodel3(0.1, r=2.0, uc=0.8, ru=32.0, wpb=8), 4, 4, cfg)
    assert three < two


def test_predict3_reduces_to_predict():
    cfg = _cfg(L0=220.0)
    a2 = O.predict(O.kmodel(0.1, r=2.0, ipb=900, wpb=4), 4, 16, O.kmodel(0.02, r=1.0, ipb=5000, wpb=8), 4, 8, 4, cfg)
    a3 = O.predict3(O.kmodel3(0.1, r=2.0, ipb=900, wpb=4), 4, 16, O.kmodel3(0.02, r=1.0, ipb=5000, wpb=8), 4, 8, 4,
                    cfg)
    assert a2.status == 0 and a3.status == 0
    for f in ("ipc1", "ipc2", "solo1", "solo2", "cp", "dT"):
        assert abs(getattr(a2, f) - getattr(a3, f)) <= 1e-9 * max(1.0, abs(getattr(a2, f))), f


@pytest.mark.parametrize("g,rm,uc", [(2, 0.3, 0.5), (4, 0.1, 1.0), (3, 0.5, 0.0)])
def test_units_w1_closed_form(g, rm, uc):
    """Block granularity (R13): one unit of g warps.  Ready: the round lasts g cycles and issues
    g instructions; idle: the round lasts 1 cycle with g*r (g*ru) requests outstanding, so
    IPC = g / (g + Rm(1-uc) L_c + Rm uc L_u)."""
    L0, a0, B, r, ru = 30.0, 1.0, 0.5, 2.0, 9.0
    cfg = _cfg(L0=L0, a0=a0, B=B, W=g)
    Lc = L0 + a0 * g * r / B
    Lu = L0 + a0 * g * ru / B + a0 * (ru - r) / B
    expect = g / (g + rm * (1 - uc) * Lc + rm * uc * Lu)
    P, R = O.build3(O.kmodel3(rm, r=r, uc=uc, ru=ru, g=g), 1, cfg)
    assert abs(O.ipc3(1, O.stationary(P), R, g1=g) - expect) < 1e-13


def test_units_g1_is_warp_model():
    cfg = _cfg()
    k1 = O.kmodel3(0.2, r=2.0, uc=0.4, ru=12.0, wpb=8, ipb=700)
    k2 = O.kmodel3(0.05, r=1.0, uc=0.0, ru=1.0, wpb=4, ipb=3000)
    a = O.predict3(k1, 2, 8, k2, 4, 16, 4, cfg)
    k1.g = 1
    b = O.predict3(k1, 2, 8, k2, 4, 16, 4, cfg)
    assert a.status == 0 and abs(a.cp - b.cp) < 1e-15


def test_units_monte_carlo():
    """Units of g = 2 warps simulated as g-instruction super-warps (independent of the chain)."""
    g, W = 2, 3
    k = dict(rm=0.3, r=2.0, uc=0.5, ru=10.0)
    L0, a0, B = 40.0, 1.0, 2.0
    cfg = _cfg(L0=L0, a0=a0, B=B, W=g * W)
    P, R = O.build3(O.kmodel3(k["rm"], r=k["r"], uc=k["uc"], ru=k["ru"], g=g), W, cfg)
    model = O.ipc3(W, O.stationary(P), R, g1=g)
    rng = np.random.default_rng(9)
    st = np.zeros(W, np.int8)
    nb, per = 50, 1200
    ib, cb = np.zeros(nb), np.zeros(nb)
    for bi in range(nb):
        inst = cyc = 0.0
        for _ in range(per):
            ready = int((st == 0).sum())
            Rr = max(g * ready, 1)
            n = g * (float((st == 1).sum()) * k["r"] + float((st == 2).sum()) * k["ru"])
            Lc = L0 + a0 * n / B
            Lu = Lc + a0 * (k["ru"] - k["r"]) / B
            x = rng.random(W)
            new = st.copy()
            rd = st == 0
            inst += g * float(rd.sum())
            new[rd & (x < k["rm"] * (1 - k["uc"]))] = 1
            new[rd & (x >= k["rm"] * (1 - k["uc"])) & (x < k["rm"])] = 2
            new[(st == 1) & (x < min(1.0, Rr / Lc))] = 0
            new[(st == 2) & (x < min(1.0, Rr / Lu))] = 0
            st = new
            cyc += Rr
        ib[bi], cb[bi] = inst, cyc
    mc = ib.sum() / cb.sum()
    sig = np.std(ib / cb, ddof=1) / math.sqrt(nb)
    assert abs(mc - model) <= 3.5 * sig + 1e-4, (mc, model, sig)

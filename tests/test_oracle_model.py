"""Pins of the oracle's Markov model (oracle/model.c) against what the paper and mathematics fix.

Each test pins the oracle to something other than itself: closed forms of the two-state chain,
a textbook special case (independent warps -> binomial), invariants (row sums, stationarity,
lumpability, symmetry), a proven bound, a per-warp Monte Carlo simulation of the round process
that shares nothing with the linear algebra, and power iteration as an independent solver.
"""
import math

import numpy as np
import pytest

import oracle as O


def _golden_examples():
    rows = {}
    for line in open(__file__.replace("test_oracle_model.py", "golden/model_worked_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        f = line.split()
        rows[f[0]] = f[1:]
    return rows


def test_w1_closed_form_golden():
    """P:825-921 with W=1: IPC = 1/(1+Rm L); Rm=1, L=9 -> pi=(0.1,0.9), IPC=0.1."""
    g = _golden_examples()
    for case in ("w1_a", "w1_b"):
        W, rm, L, p0, p1, ipc = g[case]
        cfg = O.smcfg(L0=float(L), a0=0.0, W=int(W))
        P, R = O.build_homog(O.kmodel(float(rm)), int(W), cfg)
        pi = O.stationary(P)
        assert abs(pi[0] - float(p0)) < 1e-12 and abs(pi[1] - float(p1)) < 1e-12
        assert abs(O.ipc_homog(1, pi) - float(ipc)) < 1e-12


@pytest.mark.parametrize("rm", [0.01, 0.05, 0.1, 0.2, 0.3, 0.5, 0.7, 0.9, 1.0])
@pytest.mark.parametrize("L", [2.5, 9.0, 40.0, 400.0])
def test_w1_closed_form_grid(rm, L):
    cfg = O.smcfg(L0=L, a0=0.0, W=1)
    P, _ = O.build_homog(O.kmodel(rm), 1, cfg)
    assert abs(O.ipc_homog(1, O.stationary(P)) - 1.0 / (1.0 + rm * L)) < 1e-12


@pytest.mark.parametrize("W", [1, 2, 4, 8, 12, 16, 24])
def test_rm_zero_ipc_one(W):
    """Rm = 0: no warp ever stalls, gamma_W = 0, Eq.4 gives IPC = 1 exactly."""
    cfg = O.smcfg(L0=300.0, B=1.0, a0=5.0, W=W)
    P, _ = O.build_homog(O.kmodel(0.0), W, cfg)
    assert abs(O.ipc_homog(W, O.stationary(P)) - 1.0) < 1e-12


def _rand_cfgs(n, seed=0):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        W = int(rng.integers(1, 17))
        cfg = O.smcfg(L0=float(rng.uniform(W + 5, 900)), B=float(rng.uniform(0.2, 4)),
                      a0=float(rng.uniform(0, 3)), b0=float(rng.uniform(0, 50)), W=16)
        yield W, O.kmodel(float(rng.uniform(0, 1)), r=float(rng.uniform(1, 32))), cfg


def test_rows_stochastic_and_stationary():
    """Every built matrix is row-stochastic (<=1e-12, entries in [0,1]); the LU pi satisfies
    pi P = pi to 1e-12, pi >= 0, sum 1; power iteration (independent solver) agrees."""
    for W, k, cfg in _rand_cfgs(120):
        P, _ = O.build_homog(k, W, cfg)
        assert np.all(P >= -1e-15) and np.all(P <= 1 + 1e-15)
        assert np.max(np.abs(P.sum(1) - 1)) < 1e-12
        pi = O.stationary(P)
        assert np.max(np.abs(pi @ P - pi)) < 1e-12
        assert pi.min() > -1e-14 and abs(pi.sum() - 1) < 1e-12
        Q = 0.5 * (P + np.eye(W + 1))            # lazy chain: same pi, aperiodic
        v = np.full(W + 1, 1.0 / (W + 1))
        for _ in range(200000):
            v2 = v @ Q
            if np.max(np.abs(v2 - v)) < 1e-15:
                break
            v = v2
        assert np.max(np.abs(v - pi)) < 1e-9


def test_joint_rows_stochastic():
    rng = np.random.default_rng(3)
    for _ in range(60):
        w1 = int(rng.integers(1, 9)); w2 = int(rng.integers(1, 17 - w1))
        cfg = O.smcfg(L0=float(rng.uniform(30, 900)), B=float(rng.uniform(0.2, 4)),
                      a0=float(rng.uniform(0, 3)), W=16)
        k1 = O.kmodel(float(rng.uniform(0, 1)), r=float(rng.uniform(1, 32)))
        k2 = O.kmodel(float(rng.uniform(0, 1)), r=float(rng.uniform(1, 32)))
        P, _ = O.build_joint(k1, w1, k2, w2, cfg)
        assert np.max(np.abs(P.sum(1) - 1)) < 1e-12 and P.min() >= -1e-15
        pi = O.stationary(P)
        assert np.max(np.abs(pi @ P - pi)) < 1e-12


@pytest.mark.parametrize("W,rm,q", [(1, 0.3, 0.1), (5, 0.2, 0.05), (16, 0.1, 1 / 80), (16, 0.9, 0.5)])
def test_binomial_special_case(W, rm, q):
    """With a state-independent P_ir = q every warp is an independent two-state chain, so the
    idle count is Binomial(W, Rm/(Rm+q)) (textbook); pins the Eq.2 convolution (R3)."""
    cfg = O.smcfg(W=W, pir_mode=1, const_q=q)
    P, _ = O.build_homog(O.kmodel(rm), W, cfg)
    pi = O.stationary(P)
    p = rm / (rm + q)
    ref = np.array([math.comb(W, i) * p**i * (1 - p) ** (W - i) for i in range(W + 1)])
    assert np.max(np.abs(pi - ref)) < 1e-13


def test_ipc_bound_constant_latency():
    """Proven bound for constant L: IPC <= min(1, W/(1 + Rm L)) (SURVEY §8(c) pins)."""
    rng = np.random.default_rng(5)
    for _ in range(80):
        W = int(rng.integers(1, 17)); rm = float(rng.uniform(0.01, 1)); L = float(rng.uniform(W + 1, 1000))
        P, _ = O.build_homog(O.kmodel(rm), W, O.smcfg(L0=L, a0=0.0, W=W))
        ipc = O.ipc_homog(W, O.stationary(P))
        assert ipc <= min(1.0, W / (1 + rm * L)) + 1e-12


@pytest.mark.parametrize("W", [4, 8, 12, 16])
def test_lumpability(W):
    """Identical kernels split (w1, w2): lumping joint states by p+q gives the homogeneous chain
    (matrix level, 1e-12) and C = homogeneous IPC at W = w1 + w2 (1e-12), with L depending on
    the total outstanding requests."""
    k = O.kmodel(0.15, r=4.0)
    cfg = O.smcfg(L0=200.0, B=2.0, a0=1.5, b0=10.0, W=16)
    Ph, _ = O.build_homog(k, W, cfg)
    ipc_h = O.ipc_homog(W, O.stationary(Ph))
    for w1 in range(1, W):
        w2 = W - w1
        P, R = O.build_joint(k, w1, k, w2, cfg)
        # lump: from any (p,q) with p+q = i, total mass into {p'+q' = j} equals Ph[i, j]
        for p in range(w1 + 1):
            for q in range(w2 + 1):
                s = p * (w2 + 1) + q
                lumped = np.zeros(W + 1)
                for pp in range(w1 + 1):
                    for qq in range(w2 + 1):
                        lumped[pp + qq] += P[s, pp * (w2 + 1) + qq]
                assert np.max(np.abs(lumped - Ph[p + q])) < 1e-12
        _, _, c = O.ipc_joint(w1, w2, O.stationary(P), R)
        assert abs(c - ipc_h) < 1e-12


def test_symmetry():
    k1, k2 = O.kmodel(0.3, r=2.0), O.kmodel(0.05, r=8.0)
    cfg = O.smcfg(L0=300.0, B=1.0, a0=2.0, W=16)
    P, R = O.build_joint(k1, 6, k2, 10, cfg)
    a1, a2, _ = O.ipc_joint(6, 10, O.stationary(P), R)
    P, R = O.build_joint(k2, 10, k1, 6, cfg)
    b1, b2, _ = O.ipc_joint(10, 6, O.stationary(P), R)
    assert abs(a1 - b2) < 1e-12 and abs(a2 - b1) < 1e-12
    P, R = O.build_joint(k1, 8, k1, 8, cfg)
    x1, x2, _ = O.ipc_joint(8, 8, O.stationary(P), R)
    assert abs(x1 - x2) < 1e-12


def test_cp_unit_checks():
    """Eq.1 unit values."""
    assert O.cp([1.0, 1.0], [1.0, 1.0]) == 0.5
    assert O.cp([0.5, 0.5], [1.0, 1.0]) == 0.0
    assert O.cp([1.0], [1.0]) == 0.0


def _simulate(ws, rms, rs, cfg, rounds, seed, pis=None):
    """Per-warp Monte Carlo of the round process: each ready warp issues one
    instruction and then stalls with probability Rm; each idle warp returns with probability
    P_ir = min(1, R/L) evaluated in the current state; time advances by the round duration
    R = max(#ready, 1).  Returns long-run instructions/cycle and batch-means sigma."""
    rng = np.random.default_rng(seed)
    idle = [np.zeros(w, bool) for w in ws]
    nb = 50
    per = rounds // nb
    inst_b, cyc_b = np.zeros(nb), np.zeros(nb)
    for b in range(nb):
        inst = cyc = 0.0
        for _ in range(per):
            nidle = [int(x.sum()) for x in idle]
            ready = sum(w - n for w, n in zip(ws, nidle))
            R = max(ready, 1)
            if pis:   # one pipe shared by all simulated kernels (R26)
                R = max(R, sum((w - n) / p for w, n, p in zip(ws, nidle, pis)))
            n_out = sum(n * r for n, r in zip(nidle, rs))
            L = O.latency(cfg, n_out, sum(nidle))
            pir = min(1.0, R / L)
            for k in range(len(ws)):
                u = rng.random(ws[k])
                was_idle = idle[k]
                inst += float((~was_idle).sum())
                idle[k] = np.where(was_idle, u >= pir, u < rms[k])
            cyc += R
        inst_b[b], cyc_b[b] = inst, cyc
    ipc = inst_b.sum() / cyc_b.sum()
    sig = np.std(inst_b / cyc_b, ddof=1) / math.sqrt(nb)
    return ipc, sig


@pytest.mark.parametrize("W,rm,L", [(8, 0.3, 50.0), (16, 0.1, 80.0), (1, 0.5, 10.0), (4, 0.2, 20.0)])
def test_monte_carlo_homogeneous(W, rm, L):
    cfg = O.smcfg(L0=L, a0=0.0, W=W)
    P, _ = O.build_homog(O.kmodel(rm), W, cfg)
    model = O.ipc_homog(W, O.stationary(P))
    mc, sig = _simulate([W], [rm], [1.0], cfg, 100000, seed=W)
    assert abs(mc - model) <= 3.5 * sig + 1e-4, (mc, model, sig)


def test_monte_carlo_joint():
    cfg = O.smcfg(L0=120.0, B=1.0, a0=2.0, W=16)
    k1, k2 = O.kmodel(0.25, r=2.0), O.kmodel(0.05, r=1.0)
    P, R = O.build_joint(k1, 6, k2, 10, cfg)
    a, b, c = O.ipc_joint(6, 10, O.stationary(P), R)
    mc, sig = _simulate([6, 10], [0.25, 0.05], [2.0, 1.0], cfg, 100000, seed=11)
    assert abs(mc - c) <= 3.5 * sig + 1e-4, (mc, c, sig)


def test_survey_scratch_values():
    """Cross-check values computed under readings R1-R7 by an independent scratch script
    (SURVEY §8(c) 'Scratch cross-check values'; 12 significant digits)."""
    def homog(W, rm, L0, a0):
        cfg = O.smcfg(L0=L0, B=1.0, a0=a0, W=16)
        P, _ = O.build_homog(O.kmodel(rm, r=1.0), W, cfg)
        return O.ipc_homog(W, O.stationary(P))
    assert abs(homog(16, 0.1, 80.0, 0.0) - 0.996182773483) < 1e-11
    assert abs(homog(16, 0.05, 400.0, 4.0) - 0.634428535579) < 1e-11
    assert abs(homog(8, 0.3, 50.0, 0.0) - 0.481613332960) < 1e-11
    s1, s2 = homog(16, 0.25, 300.0, 20.0), homog(16, 0.02, 300.0, 20.0)
    assert abs(s1 - 0.102855393019) < 1e-11 and abs(s2 - 0.960397950576) < 1e-11
    cfg = O.smcfg(L0=300.0, B=1.0, a0=20.0, W=16)
    P, R = O.build_joint(O.kmodel(0.25), 8, O.kmodel(0.02), 8, cfg)
    a, b, c = O.ipc_joint(8, 8, O.stationary(P), R)
    assert abs(a - 0.053138785523) < 1e-11 and abs(b - 0.569158160684) < 1e-11
    assert abs(c - 0.622296946207) < 1e-11
    assert abs(O.cp([a, b], [s1, s2]) - 0.098500773047) < 1e-11
    cfg = O.smcfg(L0=100.0, a0=0.0, W=16)
    P, R = O.build_joint(O.kmodel(0.5), 2, O.kmodel(0.01), 6, cfg)
    a, b, c = O.ipc_joint(2, 6, O.stationary(P), R)
    assert abs(a - 0.035643329673) < 1e-11 and abs(b - 0.963965632837) < 1e-11
    assert abs(c - 0.999608962510) < 1e-11
    s1, s2 = homog(16, 0.5, 100.0, 0.0), homog(16, 0.01, 100.0, 0.0)
    assert abs(O.cp([a, b], [s1, s2]) - 0.072696509857) < 1e-11


def test_predict_consistency():
    """or_predict composes the pieces: joint IPCs, solo IPCs at b_max, CP (Eq.1), dT (Eq.8)."""
    cfg = O.smcfg(L0=300.0, B=1.0, a0=2.0, W=16)
    k1, k2 = O.kmodel(0.3, r=2.0, ipb=5000.0, wpb=8), O.kmodel(0.02, r=1.0, ipb=20000.0, wpb=4)
    r = O.predict(k1, 4, 8, k2, 8, 16, 4, cfg)
    assert r.status == 0
    s1, _ = O.solo_ipc(k1, 8, 4, cfg)
    s2, _ = O.solo_ipc(k2, 16, 4, cfg)
    assert r.solo1 == s1 and r.solo2 == s2
    assert abs(r.cp - O.cp([r.ipc1, r.ipc2], [s1, s2])) < 1e-15
    assert abs(r.dT - abs(5000 * 4 / r.ipc1 - 20000 * 8 / r.ipc2)) < 1e-9 * r.dT
    assert O.predict(k1, 8, 8, k2, 8, 16, 4, cfg).status == 2      # 16 + 8 warps > W_v


@pytest.mark.parametrize("W", [1, 3, 8, 16])
@pytest.mark.parametrize("pi", [1.0, 0.68, 0.3])
def test_pipe_ceiling_rm_zero(W, pi):
    """R26: with no memory stalls every round issues W instructions in W/pi cycles: IPC = pi."""
    P, R = O.build_homog(O.kmodel(0.0, pi=pi, pipe=1), W, O.smcfg(L0=300.0, W=16))
    assert abs(O.ipc_homog(W, O.stationary(P), R) - pi) < 1e-12


@pytest.mark.parametrize("rm,L,pi", [(0.5, 10.0, 0.5), (1.0, 9.0, 0.25), (0.05, 200.0, 0.7)])
def test_pipe_ceiling_w1_closed_form(rm, L, pi):
    """R26 with W=1, constant L: the two-state balance g1 = g0 Rm L is unchanged and the ready
    round lasts 1/pi cycles, so IPC = 1/(1/pi + Rm L) = pi/(1 + pi Rm L)."""
    P, R = O.build_homog(O.kmodel(rm, pi=pi, pipe=2), 1, O.smcfg(L0=L, a0=0.0, W=1))
    assert abs(O.ipc_homog(1, O.stationary(P), R) - pi / (1 + pi * rm * L)) < 1e-12


@pytest.mark.parametrize("W", [4, 8, 12])
def test_pipe_ceiling_lumpability(W):
    """Identical kernels share their pipe: the split joint chain lumps to the homogeneous one."""
    k = O.kmodel(0.1, r=4.0, pi=0.6, pipe=1)
    cfg = O.smcfg(L0=200.0, B=2.0, a0=1.5, W=16)
    Ph, Rh = O.build_homog(k, W, cfg)
    ipc_h = O.ipc_homog(W, O.stationary(Ph), Rh)
    for w1 in range(1, W):
        P, R = O.build_joint(k, w1, k, W - w1, cfg)
        assert abs(O.ipc_joint(w1, W - w1, O.stationary(P), R)[2] - ipc_h) < 1e-12


def test_pipe_ceiling_monte_carlo():
    """Round process with pipe-bound rounds (R = max(#ready/pi, 1)) simulated per warp."""
    cfg = O.smcfg(L0=60.0, a0=0.0, W=8)
    P, R = O.build_homog(O.kmodel(0.2, pi=0.5, pipe=1), 8, cfg)
    model = O.ipc_homog(8, O.stationary(P), R)
    mc, sig = _simulate([8], [0.2], [1.0], cfg, 100000, seed=3, pis=[0.5])
    assert abs(mc - model) <= 3.5 * sig + 1e-4, (mc, model, sig)


def _simulate_pipes(ws, rms, rs, pis, pipes, cfg, rounds, seed):
    """Per-warp Monte Carlo of the R26 round for two kernels written from the reading's prose
    (R26), not from model.c: every ready warp issues once, so the round lasts at least
    #ready cycles; a kernel on a pipe of ceiling pi needs ready_k/pi_k cycles of that pipe; pipes
    are separate resources, so kernels on the same pipe queue behind each other (their pipe times
    add) and kernels on different pipes overlap.  Returns per-kernel instructions/cycle and
    batch-means sigmas."""
    rng = np.random.default_rng(seed)
    idle = [np.zeros(w, bool) for w in ws]
    nb = 50
    per = rounds // nb
    inst_b, cyc_b = np.zeros((nb, len(ws))), np.zeros(nb)
    for b in range(nb):
        for _ in range(per):
            nidle = [int(x.sum()) for x in idle]
            ready = [w - n for w, n in zip(ws, nidle)]
            busy = {}
            for rk, pk, pp in zip(ready, pis, pipes):
                busy[pp] = busy.get(pp, 0.0) + rk / pk      # cycles each pipe is busy this round
            R = max([float(sum(ready)), 1.0] + list(busy.values()))
            L = O.latency(cfg, sum(n * r for n, r in zip(nidle, rs)), sum(nidle))
            pir = min(1.0, R / L)
            for k in range(len(ws)):
                u = rng.random(ws[k])
                inst_b[b, k] += ready[k]
                idle[k] = np.where(idle[k], u >= pir, u < rms[k])
            cyc_b[b] += R
    ipc = inst_b.sum(0) / cyc_b.sum()
    sig = np.std(inst_b / cyc_b[:, None], axis=0, ddof=1) / math.sqrt(nb)
    return ipc, sig


@pytest.mark.parametrize("same_pipe", [False, True])
def test_pipe_ceiling_two_kernels_monte_carlo(same_pipe):
    """R26's joint round for two kernels with different ceilings, on different pipes (rounds
    max(r1 + r2, r1/p1, r2/p2)) and on one shared pipe (max(r1 + r2, r1/p1 + r2/p2)): per-kernel
    joint IPCs (Eq.5-6) against the simulated round process.  The ceilings are chosen so the pipe
    term binds most rounds and the two rules differ by ~40 %, so confusing them, dropping a term
    or swapping the kernels' ceilings fails."""
    cfg = O.smcfg(L0=90.0, B=1.0, a0=1.0, W=16)
    p1, p2 = 0.3, 0.5
    k1 = O.kmodel(0.06, r=2.0, pi=p1, pipe=1)
    k2 = O.kmodel(0.12, r=1.0, pi=p2, pipe=1 if same_pipe else 2)
    w1, w2 = 6, 7
    P, R = O.build_joint(k1, w1, k2, w2, cfg)
    a, b, _ = O.ipc_joint(w1, w2, O.stationary(P), R)
    mc, sig = _simulate_pipes([w1, w2], [0.06, 0.12], [2.0, 1.0], [p1, p2], [1, 1 if same_pipe else 2],
                              cfg, 60000, seed=21 + same_pipe)
    assert abs(mc[0] - a) <= 3.5 * sig[0] + 1e-4, (mc, a, b, sig)
    assert abs(mc[1] - b) <= 3.5 * sig[1] + 1e-4, (mc, a, b, sig)
    # the two readings are far apart at these parameters (the test can tell them apart)
    k2o = O.kmodel(0.12, r=1.0, pi=p2, pipe=2 if same_pipe else 1)
    Po, Ro = O.build_joint(k1, w1, k2o, w2, cfg)
    ao, bo, _ = O.ipc_joint(w1, w2, O.stationary(Po), Ro)
    assert abs(ao + bo - a - b) > 20 * (sig[0] + sig[1])


def test_reducible_chain_rejected():
    """R22: Rm=1 with P_ir clamped to 1 makes the chain an involution; the guard L > W rejects."""
    with pytest.raises(ValueError):
        O.build_homog(O.kmodel(1.0), 16, O.smcfg(L0=10.0, a0=0.0, W=16))

"""GPU parity of the batched Markov model (kl_predict) and of FindCoSchedule's decision
(kl_decide: device-fused selection on a cache miss, host selection on a hit) against the oracle."""
import numpy as np
import pytest

import oracle as O
import paper_1303_5164_b200 as K

pytestmark = pytest.mark.gpu

CFG = dict(L0=700.0, B=0.3, a0=1.0, b0=20.0)


def _rand_profiles(rng):
    profs = {}
    for k in K.KINDS:
        wpb = int(rng.choice([1, 2, 4, 8]))
        bmax = int(min(32, 64 // wpb, rng.integers(2, 33)))
        profs[k] = dict(rm=float(rng.uniform(0.001, 0.6)), r=float(rng.uniform(1, 32)),
                        ipb=float(rng.uniform(100, 50000)), pur=float(rng.uniform(0, 1)),
                        mur=float(rng.uniform(0, 0.3)), wpb=wpb, regs=int(rng.choice([16, 32, 48, 64])),
                        smem=int(rng.choice([0, 2048, 16384])), tmem=0, bmax=bmax, m_min=1,
                        ipc_max=float(rng.choice([1.0, rng.uniform(0.2, 1.0)])), pipe=int(rng.integers(0, 3)))
    return profs


def _ctx(profs, **kw):
    K.build()
    return K.Context(device=0, profiles=profs, **CFG, **kw)


def test_predict_matches_oracle():
    rng = np.random.default_rng(0)
    worst = 0.0
    for rep in range(3):
        profs = _rand_profiles(rng)
        ctx = _ctx(profs)
        cfg = O.smcfg(W=16, **CFG)
        cands = []
        for _ in range(300):
            k1, k2 = rng.choice(K.KINDS, 2)
            p1, p2 = profs[k1], profs[k2]
            l1, l2 = O.levels(p1), O.levels(p2)
            if not l1 or not l2:
                continue
            b1, b2 = int(rng.choice(l1)), int(rng.choice(l2))
            if b1 * p1["wpb"] + b2 * p2["wpb"] > 64:
                continue
            cands.append((str(k1), str(k2), b1, b2))
        preds = ctx.predict(cands)
        for (k1, k2, b1, b2), g in zip(cands, preds):
            p1, p2 = profs[k1], profs[k2]
            r = O.predict(O.kmodel_of(p1), b1, O.solo_b(p1), O.kmodel_of(p2), b2, O.solo_b(p2), 4, cfg)
            assert g.status == r.status, (k1, k2, b1, b2, g.status, r.status)
            if r.status:
                continue
            for f in ("ipc1", "ipc2", "c", "solo1", "solo2", "cp"):
                e = abs(getattr(g, f) - getattr(r, f))
                worst = max(worst, e)
                assert e <= 1e-9, (f, k1, k2, b1, b2, getattr(g, f), getattr(r, f))
            # dT is a difference of two per-wave times: compare relative to the terms (Eq.8)
            terms = max(p1["ipb"] * b1 / r.ipc1, p2["ipb"] * b2 / r.ipc2)
            assert abs(g.dT - r.dT) <= 1e-9 * terms
        ctx.close()
    print("max abs model error vs oracle:", worst)


def _decide_both(ctx):
    d1 = ctx.decide()          # cold cache: device model + fused device selection
    d2 = ctx.decide()          # warm cache: host selection
    return d1, d2


def test_solo_queries_match_oracle():
    """b2 = 0 asks the device model for k1 alone at b1 (used by the calibration fit)."""
    rng = np.random.default_rng(11)
    profs = _rand_profiles(rng)
    ctx = _ctx(profs)
    cfg = O.smcfg(W=16, **CFG)
    cands = [(k, k, b, 0) for k in K.KINDS for b in O.levels(profs[k])]
    for (k, _, b, _), g in zip(cands, ctx.predict(cands)):
        ref, st = O.solo_ipc(O.kmodel_of(profs[k]), b, 4, cfg)
        assert g.status == st
        if st == 0:
            assert abs(g.ipc1 - ref) < 1e-9, (k, b, g.ipc1, ref)
    ctx.close()


def test_decisions_match_oracle():
    rng = np.random.default_rng(7)
    n_cmp = 0
    for rep in range(12):
        profs = _rand_profiles(rng)
        cp_min = float(rng.choice([0.0, 0.02]))
        rule = int(rep % 2)
        ctx = _ctx(profs, alpha_p=float(rng.choice([0.0, 0.2, 0.4])), alpha_m=float(rng.choice([0.0, 0.05, 0.1])),
                   cp_min=cp_min, split_rule=rule)
        n = int(rng.integers(1, 9))
        kinds = [str(k) for k in rng.choice([k for k in K.KINDS if k != "MM"], n)]
        pend = []
        for k in kinds:
            kid = ctx.submit(k, 1000, K.ARGS[K.KIND_ID[k]]())
            pend.append({"kind": k, "blocks": 1000, "id": kid})
        d1, d2 = _decide_both(ctx)
        ref = O.find_co_schedule(pend, profs, O.smcfg(W=16, **CFG), ap=ctx.config.alpha_p,
                                 am=ctx.config.alpha_m, cp_min=cp_min, split_rule=rule)
        for d in (d1, d2):
            assert bool(d.solo) == bool(ref["solo"]), (kinds, d.solo, ref["solo"])
            assert d.id1 == pend[ref["ia"]]["id"]
            if not ref["solo"]:
                assert d.id2 == pend[ref["ib"]]["id"]
                assert (d.b1, d.b2) == (ref["b1"], ref["b2"])
                assert abs(d.cp - ref["cp"]) < 1e-9
            else:
                assert d.b1 == ref["b1"]
        n_cmp += 1
        ctx.close()
    assert n_cmp == 12

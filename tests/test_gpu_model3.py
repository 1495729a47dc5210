"""GPU parity of the f1 general model (csrc/kl_model3.cu): three-state coalesced/uncoalesced
chains (reading R27) and thread blocks as the modelling unit (R13),
through kl_predict and kl_decide, against the oracle (oracle/model3.c, dense LU)."""
import numpy as np
import pytest

import oracle as O
import paper_1303_5164_b200 as K
from test_gpu_model import CFG, _rand_profiles

pytestmark = pytest.mark.gpu


def _profs3(rng):
    profs = _rand_profiles(rng)
    for k, p in profs.items():
        if rng.random() < 0.5:
            p["uc"] = float(rng.uniform(0.05, 1.0))
            p["ru"] = p["r"] + float(rng.uniform(0.0, 24.0))
    return profs


def _cands(rng, profs, n, max_states=None, states=3, gran=0):
    out = []
    for _ in range(n * 4):
        k1, k2 = (str(x) for x in rng.choice(K.KINDS, 2))
        p1, p2 = profs[k1], profs[k2]
        l1, l2 = O.levels(p1), O.levels(p2)
        if not l1 or not l2:
            continue
        b1, b2 = int(rng.choice(l1)), int(rng.choice(l2))
        if b1 * p1["wpb"] + b2 * p2["wpb"] > 64:
            continue
        if max_states:
            def ns(p, b):
                m = O.kmodel3_of(p, states, gran)
                w = b * p["wpb"] // 4
                u = max(1, w // m.g)
                return (u + 1) * (u + 2) // 2 if m.uc > 0 else u + 1
            if ns(p1, b1) * ns(p2, b2) > max_states or ns(p1, O.solo_b(p1)) > max_states or ns(p2, O.solo_b(p2)) > max_states:
                continue
        out.append((k1, k2, b1, b2))
        if len(out) == n:
            break
    return out


def _check(ctx, profs, cands, states, gran):
    cfg = O.smcfg(W=16, **CFG)
    worst = 0.0
    for (k1, k2, b1, b2), g in zip(cands, ctx.predict(cands)):
        p1, p2 = profs[k1], profs[k2]
        r = O.predict_cfg(p1, b1, p2, b2, cfg, 4, states, gran)
        assert g.status == r.status, (k1, k2, b1, b2, g.status, r.status)
        if r.status:
            continue
        for f in ("ipc1", "ipc2", "c", "solo1", "solo2", "cp"):
            e = abs(getattr(g, f) - getattr(r, f))
            worst = max(worst, e)
            assert e <= 1e-9, (f, k1, k2, b1, b2, getattr(g, f), getattr(r, f))
        terms = max(p1["ipb"] * b1 / r.ipc1, p2["ipb"] * b2 / r.ipc2)
        assert abs(g.dT - r.dT) <= 1e-9 * terms
    return worst


@pytest.mark.parametrize("seed", [0, 1])
def test_three_state_predict_matches_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    profs = _profs3(rng)
    ctx = K.Context(device=0, profiles=profs, model_states=3, **CFG)
    cands = _cands(rng, profs, 60, max_states=600)
    assert len(cands) >= 20
    print("worst", _check(ctx, profs, cands, 3, 0))
    ctx.close()


def test_block_granularity_matches_oracle():
    rng = np.random.default_rng(7)
    profs = _profs3(rng)
    ctx = K.Context(device=0, profiles=profs, model_states=3, granularity=1, **CFG)
    cands = _cands(rng, profs, 60, max_states=600, gran=1)
    print("worst", _check(ctx, profs, cands, 3, 1))
    ctx.close()


def test_large_three_state_chain():
    """Both kernels three-state at 8 + 8 warps: 45 x 45 = 2025 joint states (global scratch)."""
    profs = _rand_profiles(np.random.default_rng(3))
    for k in ("PC", "SPMV"):
        profs[k].update(wpb=8, bmax=8, rm=0.2, r=2.0, uc=0.6, ru=16.0, regs=32, smem=0, ipc_max=1.0, pipe=0)
    ctx = K.Context(device=0, profiles=profs, model_states=3, **CFG)
    _check(ctx, profs, [("PC", "SPMV", 4, 4)], 3, 0)
    ctx.close()


def test_general_kernel_reduces_to_two_state():
    """model_states = 3 with no uncoalesced kind runs the general kernel's two-state path: the
    same predictions as the shared-memory two-state kernel."""
    rng = np.random.default_rng(5)
    profs = _rand_profiles(rng)
    a = K.Context(device=0, profiles=profs, **CFG)
    pb = {k: dict(v) for k, v in profs.items()}
    pb["MATADD"]["uc"] = 0.5      # one three-state kind in the table selects the general kernel
    b = K.Context(device=0, profiles=pb, granularity=0, model_states=3, **CFG)
    cands = [c for c in _cands(rng, profs, 120) if "MATADD" not in c[:2]][:80]
    pa, pb = a.predict(cands), b.predict(cands)
    for x, y in zip(pa, pb):
        assert x.status == y.status
        if x.status == 0:
            assert abs(x.cp - y.cp) < 1e-10 and abs(x.ipc1 - y.ipc1) < 1e-10
    a.close()
    b.close()


def test_three_state_decisions_match_oracle():
    rng = np.random.default_rng(21)
    for rep in range(6):
        profs = _profs3(rng)
        gran = rep % 2
        ctx = K.Context(device=0, profiles=profs, model_states=3, granularity=gran, alpha_p=0.0, alpha_m=0.0, **CFG)
        kinds = [str(k) for k in rng.choice([k for k in K.KINDS if k != "MM"], int(rng.integers(2, 6)))]
        pend = []
        for k in kinds:
            kid = ctx.submit(k, 1000, K.ARGS[K.KIND_ID[k]]())
            pend.append({"kind": k, "blocks": 1000, "id": kid})
        d = ctx.decide()
        ref = O.find_co_schedule(pend, profs, O.smcfg(W=16, **CFG), ap=0.0, am=0.0, states=3, granularity=gran)
        assert bool(d.solo) == bool(ref["solo"])
        assert d.id1 == pend[ref["ia"]]["id"]
        if not ref["solo"]:
            assert d.id2 == pend[ref["ib"]]["id"] and (d.b1, d.b2) == (ref["b1"], ref["b2"])
            assert abs(d.cp - ref["cp"]) < 1e-9
        ctx.close()

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


def _args_of(kind, keep={}):
    """Descriptor args for decide-only submissions: zero structs, except MM, whose prepare step
    encodes TMA descriptors and so needs a real (small) operand set."""
    if kind != "MM":
        return 1000, K.ARGS[K.KIND_ID[kind]]()
    if "MM" not in keep:
        import kl_inputs as G
        from paper_1303_5164_b200.workload import Instance
        keep["MM"] = Instance(G.gen("MM", "small"), "cuda")
    return keep["MM"].grid, keep["MM"].args


def _bench_profiles(levels="four", bmax="hw"):
    """The calibrated B200 profile and scheduler config the bench runs (bench.load_profiles; with
    every whole-warp level and bmax="sat", b_max is the saturation occupancy, R31)."""
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    return bench.load_profiles(os.path.join(root, "profiles", "kl_profile_b200.json"), levels, bmax)


@pytest.mark.parametrize("level_mode,bmax", [(1, "hw"), (0, "hw"), (0, "sat")])
@pytest.mark.parametrize("split_rule", [1, 0])
def test_decisions_match_oracle_bench_config(split_rule, level_mode, bmax):
    """The bench's decision configurations: calibrated profiles with the resource fields the
    runtime reads from the compiled kernels (MM: TMEM- and shared-memory-bound, one block per SM),
    the four C2 occupancy levels (level_mode = 1 <-> oracle mode "4"; C2) or every whole-warp level
    (level_mode = 0 <-> oracle mode "all"; C4 / C5), alpha = 0, the calibrated cp_min and both split
    rules; queues drawn from the ALL mix always holding MM.  The oracle gets the runtime-resolved
    profiles (kl_get_profile), so this compares the decision logic, not the profile plumbing."""
    K.build()
    profs, kcfg = _bench_profiles("four" if level_mode == 1 else "all", bmax)
    cfg = dict(kcfg)
    cfg.update(split_rule=split_rule, level_mode=level_mode, distinct_kinds=int(bmax == "sat"))
    rng = np.random.default_rng(23 + split_rule + 7 * level_mode)
    all_mix = ["PC", "SAD", "SPMV", "ST", "MM", "MRIQ", "BS", "TEA"]
    for rep in range(16):
        ctx = K.Context(device=0, profiles=profs, **cfg)
        resolved = {k: K.profile_dict(ctx.get_profile(k)) for k in all_mix}
        assert resolved["MM"]["bmax"] == 1 and resolved["MM"]["tmem"] > 0
        n = int(rng.integers(1, 9))
        kinds = ["MM"] + [str(k) for k in rng.choice(all_mix, n)]
        rng.shuffle(kinds)
        pend = []
        for k in kinds:
            kid = ctx.submit(k, *_args_of(k))
            pend.append({"kind": k, "blocks": 1000, "id": kid})
        d1, d2 = _decide_both(ctx)
        ocfg = O.smcfg(W=16, L0=kcfg["L0"], B=kcfg["B"], a0=kcfg.get("a0", 1.0), b0=kcfg.get("b0", 0.0))
        ref = O.find_co_schedule(pend, resolved, ocfg, ap=ctx.config.alpha_p, am=ctx.config.alpha_m,
                                 mode="4" if level_mode == 1 else "all", cp_min=ctx.config.cp_min,
                                 split_rule=split_rule, distinct_kinds=bool(ctx.config.distinct_kinds))
        for d in (d1, d2):
            assert bool(d.solo) == bool(ref["solo"]), (kinds, d.solo, ref["solo"])
            assert d.id1 == pend[ref["ia"]]["id"], (kinds, d.id1, ref)
            if not ref["solo"]:
                assert d.id2 == pend[ref["ib"]]["id"]
                assert (d.b1, d.b2) == (ref["b1"], ref["b2"]), (kinds, d.b1, d.b2, ref["b1"], ref["b2"])
                assert abs(d.cp - ref["cp"]) < 1e-9
            else:
                assert d.b1 == ref["b1"]
        ctx.close()


def test_opt_frozen_table_decisions():
    """f2 OPT path: a prediction table installed with kl_cache_put and
    model_frozen = 1 drives the decisions without the device model; they equal the oracle's
    FindCoSchedule run on the same table (its `cache` argument), and a candidate without an
    installed entry is never chosen (infeasible)."""
    K.build()
    profs, kcfg = _bench_profiles()
    rng = np.random.default_rng(31)
    all_mix = ["PC", "SAD", "SPMV", "ST", "MM", "MRIQ", "BS", "TEA"]
    for rep in range(8):
        ctx = K.Context(device=0, profiles=profs, **dict(kcfg, model_frozen=1, split_rule=rep % 2, level_mode=1))
        resolved = {k: K.profile_dict(ctx.get_profile(k)) for k in all_mix}
        # a synthetic "measured" table: random CPs over every maximal split of every kind pair,
        # with about a quarter of the candidates left out
        table, items = {}, []
        for i, a in enumerate(all_mix):
            for b in all_mix[i:]:
                for (b1, b2) in O.maximal_splits(O.B200_SM, resolved[a], resolved[b], 4, "4"):
                    if rng.random() < 0.25:
                        continue
                    i1, i2 = float(rng.uniform(0.05, 0.9)), float(rng.uniform(0.05, 0.9))
                    s1, s2 = float(rng.uniform(0.3, 1.0)), float(rng.uniform(0.3, 1.0))
                    pr = dict(ipc1=i1, ipc2=i2, c=i1 + i2, solo1=s1, solo2=s2,
                              cp=1.0 - 1.0 / (i1 / s1 + i2 / s2), dT=float(rng.uniform(0, 1e6)), status=0)
                    table[(a, b, b1, b2)] = pr
                    items.append(((a, b, b1, b2), pr))
                    if a != b:   # the runtime looks the pair up in either order
                        sw = dict(ipc1=i2, ipc2=i1, c=i1 + i2, solo1=s2, solo2=s1, cp=pr["cp"], dT=pr["dT"], status=0)
                        table[(b, a, b2, b1)] = sw
                        items.append(((b, a, b2, b1), sw))
        ctx.cache_put(items)
        kinds = [str(k) for k in rng.choice(all_mix, int(rng.integers(2, 9)))]
        pend = []
        for k in kinds:
            pend.append({"kind": k, "blocks": 1000, "id": ctx.submit(k, *_args_of(k))})
        d = ctx.decide()
        # entries the table lacks are infeasible to both sides
        cache = {key: table.get(key, dict(status=2, ipc1=0, ipc2=0, c=0, solo1=0, solo2=0, cp=0, dT=0))
                 for a in all_mix for b in all_mix
                 for (b1, b2) in O.maximal_splits(O.B200_SM, resolved[a], resolved[b], 4, "4")
                 for key in [(a, b, b1, b2)]}
        ocfg = O.smcfg(W=16, L0=kcfg["L0"], B=kcfg["B"], a0=kcfg.get("a0", 1.0), b0=kcfg.get("b0", 0.0))
        ref = O.find_co_schedule(pend, resolved, ocfg, ap=ctx.config.alpha_p, am=ctx.config.alpha_m, mode="4",
                                 cp_min=ctx.config.cp_min, split_rule=rep % 2, cache=cache)
        assert bool(d.solo) == bool(ref["solo"]), (kinds, d.solo, ref)
        assert d.id1 == pend[ref["ia"]]["id"]
        if not ref["solo"]:
            assert d.id2 == pend[ref["ib"]]["id"]
            assert (d.b1, d.b2) == (ref["b1"], ref["b2"])
            assert abs(d.cp - table[(pend[ref["ia"]]["kind"], pend[ref["ib"]]["kind"], d.b1, d.b2)]["cp"]) < 1e-12
        assert ctx.stats().model_batches == 0          # the device model never ran
        ctx.close()

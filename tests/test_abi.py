"""CPU checks of the C ABI boundary: libkl.so builds for sm_100a, loads without a GPU, exports every
symbol include/kl.h declares, the ctypes mirror matches the C struct layouts, and the host-only
logic (submit validation, slicing plans, occupancy feasibility) behaves as documented."""
import ctypes as C
import os
import re

import pytest

import kl_inputs as G
import paper_1303_5164_b200 as K

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    K.build()
    return K.lib()


def test_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "kl.h")).read()
    declared = set(re.findall(r"^\s*(?:kl_status|int|const char\*)\s+(kl_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 18
    assert declared == set(K.ABI_SYMBOLS)
    for s in declared:
        assert hasattr(L, s), s
    assert L.kl_abi_version() == 3


def test_struct_layouts_match(L):
    out = (C.c_uint32 * 32)()
    n = L.kl_struct_sizes(out, 32)
    assert n == len(K.STRUCTS)
    for i, name in enumerate(K.STRUCTS):
        assert C.sizeof(getattr(K, name)) == out[i], name


def test_kind_enum_matches_generators():
    hdr = open(os.path.join(ROOT, "include", "kl.h")).read()
    for i, k in enumerate(K.KINDS):
        assert re.search(rf"KL_{k}\s*=\s*{i}\b", hdr), k
    assert K.KINDS == G.KINDS


def _host_ctx(**kw):
    profs = {k: dict(rm=0.1, r=1.0, ipb=100.0, pur=0.1, mur=0.1, wpb=G.THREADS[k] // 32, regs=32,
                     smem=0, bmax=min(32, 64 // max(1, G.THREADS[k] // 32)), m_min=1) for k in K.KINDS}
    return K.Context(device=-1, profiles=profs, **kw)


def test_matrixadd_slicing_example(L):
    """Fig. fig:slicing: 256x256 MatrixAdd, 16x16 blocks; 8-block slices -> 32 slices."""
    ctx = _host_ctx(n_sms=148)
    a = K.ArgsMATADD(0, 0, 0, 256)
    kid = ctx.submit("MATADD", 256, a)
    p = ctx.slice(kid, blocks_per_sm=1, slice_blocks=8)
    assert (p.slice_blocks, p.n_slices) == (8, 32)
    p = ctx.slice(kid, blocks_per_sm=2)            # p% rule default: m_min = 1 wave of 2 x 148
    assert (p.slice_blocks, p.n_slices, p.waves) == (296, 1, 1)


def test_slicing_plan_p_percent_rule(L):
    ctx = _host_ctx(n_sms=14)
    ctx.set_profile("PC", dict(rm=0.2, r=32.0, ipb=700.0, pur=0.01, mur=0.14, m_min=3))
    kid = ctx.submit("PC", 16384, K.ArgsPC(0, 0, 0, 1 << 20, 10, 16384 * 256))
    p = ctx.slice(kid, blocks_per_sm=1)            # 3 waves of 1 x 14 = 42 blocks (C2050)
    assert p.slice_blocks == 42 and p.n_slices == -(-16384 // 42)


def test_submit_validation_and_infeasible(L):
    ctx = _host_ctx()
    with pytest.raises(K.KlError) as e:
        ctx.submit("PC", 0, K.ArgsPC())
    assert e.value.status == K.KL_EINVAL
    with pytest.raises(K.KlError) as e:        # wrong args struct size for the kind
        ctx.submit("PC", 10, K.ArgsBS())
    assert e.value.status == K.KL_EINVAL
    kid = ctx.submit("PC", 10, K.ArgsPC())
    with pytest.raises(K.KlError) as e:        # 9 blocks of 8 warps > 64 warps
        ctx.slice(kid, blocks_per_sm=9)
    assert e.value.status == K.KL_EINFEASIBLE and "warps" in str(e.value)
    with pytest.raises(K.KlError) as e:
        ctx.set_profile("PC", dict(rm=1.5))
    assert e.value.status == K.KL_EINVAL
    with pytest.raises(K.KlError) as e:
        ctx.slice(999, 1)
    assert e.value.status == K.KL_ENOTFOUND


def test_host_only_refuses_device_calls(L):
    ctx = _host_ctx()
    ctx.submit("BS", 10, K.ArgsBS())
    with pytest.raises(K.KlError) as e:
        ctx.sync()
    assert e.value.status == K.KL_ECUDA


def test_config_validation(L):
    """kl_create rejects an MM ring depth that is not one of its occupancy levels (R28), a
    scheduler count that does not divide the 64 warps of an SM, a distinct_kinds flag (R31b)
    other than 0 / 1 and a non-zero reserved field."""
    for bad in (dict(mm_stages=5), dict(mm_stages=1), dict(n_sched=3), dict(distinct_kinds=2),
                dict(reserved0=1)):
        with pytest.raises(K.KlError) as e:
            _host_ctx(**bad)
        assert e.value.status == K.KL_EINVAL, bad
    for ok in (0, 2, 3, 4, 6):
        _host_ctx(mm_stages=ok).close()
    for ok in (0, 1):
        _host_ctx(distinct_kinds=ok).close()

"""GPU parity of the sm_100a benchmark kernels through the C ABI (libkl.so).

For every kind at oracle-sized inputs (several tiles and a ragged tail):
  * unsliced plain launch (kl_run_plain over the whole grid) vs the oracle;
  * explicit slicing with index rectification at many slice sizes, and in a permuted
    slice order, bit-identical to the unsliced GPU result (block independence);
  * the same kernel submitted to the scheduler (persistent slice launcher, solo phase) with the
    coverage audit: every virtual block executed exactly once.
"""
import numpy as np
import pytest
import torch

import kl_inputs as G
import oracle as O
import paper_1303_5164_b200 as K
from paper_1303_5164_b200.workload import Instance
from kl_check import compare

pytestmark = pytest.mark.gpu

KINDS = ["PC", "SAD", "SPMV", "ST", "MM", "MRIQ", "BS", "TEA", "MATADD", "SYNTH"]


@pytest.fixture(scope="module")
def ctx():
    K.build()
    c = K.Context(device=0, audit=1)
    yield c
    c.close()


def _run_plain(ctx, inst, slices=None):
    for o in inst.outputs.values():
        o.fill_(0)
    if slices is None:
        ctx.run_plain(inst.kind, inst.grid, inst.args, 0)
    else:
        for off, n in slices:
            ctx.run_plain(inst.kind, inst.grid, inst.args, 0, off, n)
    torch.cuda.synchronize()
    return inst.result()


@pytest.mark.parametrize("kind", KINDS)
def test_unsliced_vs_oracle(ctx, kind):
    d = G.gen(kind, "small")
    inst = Instance(d, "cuda")
    res = _run_plain(ctx, inst)
    ref = O.run_kernel(d)
    compare(kind, res, ref)


@pytest.mark.parametrize("kind", KINDS)
def test_sliced_bit_identical(ctx, kind):
    d = G.gen(kind, "small")
    inst = Instance(d, "cuda")
    base = _run_plain(ctx, inst)
    k = inst.grid
    rng = np.random.default_rng(1)
    for s in sorted({1, 2, 3, 8, 37, max(1, k // 3), k}):
        sl = [(o, min(s, k - o)) for o in range(0, k, s)]
        res = _run_plain(ctx, inst, sl)
        for f in base:
            assert np.array_equal(res[f], base[f]), (kind, s, f)
    sl = [(o, min(5, k - o)) for o in range(0, k, 5)]
    rng.shuffle(sl)
    res = _run_plain(ctx, inst, sl)
    for f in base:
        assert np.array_equal(res[f], base[f]), (kind, "permuted", f)


@pytest.mark.parametrize("kind", KINDS)
def test_scheduler_solo_audit(ctx, kind):
    d = G.gen(kind, "small")
    inst = Instance(d, "cuda")
    base = _run_plain(ctx, inst)
    for o in inst.outputs.values():
        o.fill_(0)
    torch.cuda.synchronize()   # library lanes are non-blocking streams
    kid = ctx.submit(kind, inst.grid, inst.args, tag=7)
    ctx.sync()
    res = inst.result()
    for f in base:
        assert np.array_equal(res[f], base[f]), (kind, f)
    counts = ctx.audit(kid, inst.grid)
    assert np.all(counts == 1), (kind, counts.min(), counts.max())


def test_matrixadd_paper_slicing_example(ctx):
    """Fig. fig:slicing: 256x256 MatrixAdd as 32 slices of 8 blocks equals the unsliced kernel."""
    d = G.gen("MATADD", "small")
    inst = Instance(d, "cuda")
    res = _run_plain(ctx, inst, [(o, 8) for o in range(0, 256, 8)])
    assert np.array_equal(res["C"], (d["A"] + d["B"]).reshape(-1))


def test_laplacian_mode_exact(ctx):
    """ST with c1 = 1, c0 = 6 on an integer field is integer-exact on the GPU too."""
    d = G.gen("ST", "small", mode="int")
    inst = Instance(d, "cuda", c0=6.0, c1=1.0)
    res = _run_plain(ctx, inst)
    ref = O.run_kernel(d, c0=6.0, c1=1.0)
    assert np.array_equal(res["out"], ref["out"])


@pytest.mark.parametrize("kind,field", [("SPMV", "y"), ("MM", "C")])
def test_integer_modes_exact(ctx, kind, field):
    """Small-integer inputs make every partial sum exact in fp32: bit-exact vs the oracle."""
    d = G.gen(kind, "small", mode="int")
    inst = Instance(d, "cuda")
    res = _run_plain(ctx, inst)
    ref = O.run_kernel(d)
    assert np.array_equal(res[field], ref[field])


@pytest.mark.parametrize("num_k", [1, 7, 8, 9, 255, 256, 263, 2048])
def test_mriq_num_k_edges(ctx, num_k):
    """MRIQ's k loop: 256-point staging chunks, unrolled groups of KL_MRIQ_G = 8 (of which the last
    KL_MRIQ_P use the FMA-pipe polynomials in the experimental builds) and ragged tails, against
    the oracle; the phase range reaches |k.x| of ~48 revolutions (kx, ky, kz ~ U[-32, 32),
    x ~ U[-0.5, 0.5)).  Below 64 k-points the normwise bound has no averaging to lean on, and the
    fp32 phase t = k.x itself is off by up to ulp(|t|) (~2e-5 rad at 300 rad), so those cases draw
    k from U[-4, 4)."""
    d = G.gen("MRIQ", dict(num_x=777, num_k=num_k))
    if num_k < 64:
        for f in ("kx", "ky", "kz"):
            d[f] = (d[f] * np.float32(0.125)).astype(np.float32)
    inst = Instance(d, "cuda")
    compare("MRIQ", _run_plain(ctx, inst), O.run_kernel(d))


def test_mriq_zero_k_closed_form(ctx):
    """k = 0 for every k-point: cos = 1 and sin = 0 exactly, so Qr = sum phiMag and Qi = 0 (the
    oracle's closed-form pin), bit-exact in fp32 (fmaf(phi, 1, q) = phi + q)."""
    d = G.gen("MRIQ", dict(num_x=300, num_k=16))
    for f in ("kx", "ky", "kz"):
        d[f][:] = 0
    inst = Instance(d, "cuda")
    res = _run_plain(ctx, inst)
    acc = np.float32(0)
    for v in np.asarray(d["phimag"], np.float32):
        acc = np.float32(acc + v)
    assert np.all(np.asarray(res["qi"]) == 0)
    assert np.all(np.asarray(res["qr"]) == acc)

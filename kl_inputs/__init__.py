"""Seeded synthetic inputs for the eight Kernelet benchmark kernels (+ MatrixAdd, Synthetic).

This module is the ONE piece of code shared by the CPU oracle (`oracle/`) and the CUDA path
(`paper_1303_5164_b200/`).  It holds no arithmetic of the method: it only draws random input
bytes with numpy's PCG64 (`np.random.default_rng(seed)`) in the shapes, sizes and value
ranges of the paper's workloads (PAPER.md `tb:description`; readings R17/R18 of
SURVEY.md §8(c)).  Kernel semantics (what is computed from these inputs) live separately in
`oracle/kernels.c` (plain C) and `paper_1303_5164_b200/csrc/kl_kernels.cu` (CUDA).

Every generator returns a dict with numpy arrays (C-contiguous) and scalar params, plus the
grid size `grid_blocks` and threads per block `threads` of the paper's thread configuration,
because those define the block decomposition that slicing works on.

Size presets:
  PAPER  - tb:description sizes ("million" = 2^20, R17)
  SMALL  - sizes the oracle finishes in well under a second, spanning several tiles and a
           ragged tail (grid not a multiple of the slice size / tile).
"""
from __future__ import annotations

import numpy as np

MIB = 1 << 20

# Kind ids -- must match include/kl.h kl_kind (checked by tests/test_abi.py).
KINDS = ["PC", "SAD", "SPMV", "ST", "MM", "MRIQ", "BS", "TEA", "MATADD", "SYNTH"]
KIND_ID = {k: i for i, k in enumerate(KINDS)}

PAPER = {
    # P:1139 "Index values for 40 million accesses", 256 x 16384 threads -> H = 10 hops/thread
    "PC": dict(n_nodes=40 * MIB, n_threads=256 * 16384, hops=10),
    # P:1140 1920x1072 image, 32 x 8048 threads (8040 macroblocks padded to a multiple of 16)
    "SAD": dict(width=1920, height=1072),
    # P:1141 131072 x 81200, 16 nnz per row on average, 256 x 16384 threads (one warp per row)
    "SPMV": dict(n_rows=131072, n_cols=81200, nnz_min=8, nnz_max=24),
    # P:1142 134217728 = 512^3 points, 128 x 16384 threads (32x4 tile x 64 z-points)
    "ST": dict(nx=512, ny=512, nz=512),
    # P:1143 8192x2048 times 2048x2048
    "MM": dict(M=8192, N=2048, K=2048),
    # P:1144 2097152 elements, 256 x 8192 threads; numK free (R17 -> 2048)
    "MRIQ": dict(num_x=2 * MIB, num_k=2048),
    # P:1145 40 million options, 128 x 16384 threads (20 options per thread)
    "BS": dict(n=40 * MIB),
    # P:1146 20971520 elements (64-bit blocks), 128 x 16384 threads (10 blocks per thread)
    "TEA": dict(n=20971520),
    # P:509-530 MatrixAdd 256x256, 16x16 blocks of 16x16 threads
    "MATADD": dict(n=256),
    # SURVEY K10 "testing kernel": streaming float4 loads + c dependent FMAs
    "SYNTH": dict(n=1 << 28, fmas=4),
}

SMALL = {
    "PC": dict(n_nodes=1 << 16, n_threads=256 * 64, hops=10),          # config C1
    "SAD": dict(width=176, height=112),                                   # 11x7 = 77 macroblocks
    "SPMV": dict(n_rows=1003, n_cols=800, nnz_min=8, nnz_max=24),       # ragged last block
    "ST": dict(nx=96, ny=20, nz=136),                                     # partial tiles in y and z
    "MM": dict(M=512, N=256, K=192),
    "MRIQ": dict(num_x=10007, num_k=300),
    "BS": dict(n=128 * 20 * 64),                                          # config C1: 163840
    "TEA": dict(n=128 * 10 * 37 + 6),
    "MATADD": dict(n=256),
    "SYNTH": dict(n=256 * 4 * 4 * 37, fmas=4),
}

# Seeds per kind for the ALL-mix queue (seeds 10..17)
KIND_SEED = {"PC": 10, "SAD": 11, "SPMV": 12, "ST": 13, "MM": 14, "MRIQ": 15, "BS": 16, "TEA": 17,
             "MATADD": 18, "SYNTH": 19}

# Thread configuration (threads per block) per kind, P:1139-1146 (MM: our tcgen05 tile CTA).
THREADS = {"PC": 256, "SAD": 32, "SPMV": 256, "ST": 128, "MM": 256, "MRIQ": 256, "BS": 128,
           "TEA": 128, "MATADD": 256, "SYNTH": 256}

# Per-block work units that fix the grid decomposition (shared layout facts, not arithmetic).
SAD_MB = 16            # macroblock edge
SAD_RANGE = 16         # search offsets in [-16, 16]
SPMV_ROWS_PER_BLOCK = 8
ST_TILE = (128, 4, 32)  # x, y, z points per block (32 threads x float4 in x, 4 rows)
MM_TILE = (256, 256)   # output tile (M, N) per block (a CTA pair)
BS_PER_BLOCK = 128 * 20
TEA_PER_BLOCK = 128 * 10
MRIQ_PER_BLOCK = 256
SYNTH_F4_PER_THREAD = 4


def _cdiv(a, b):
    return -(-a // b)


def grid_blocks(kind: str, p: dict) -> int:
    """Number of thread blocks k of the kernel at the given size."""
    if kind == "PC":
        return p["n_threads"] // THREADS["PC"]
    if kind == "SAD":
        n_mb = (p["width"] // SAD_MB) * (p["height"] // SAD_MB)
        return _cdiv(n_mb, 16) * 16
    if kind == "SPMV":
        return _cdiv(p["n_rows"], SPMV_ROWS_PER_BLOCK)
    if kind == "ST":
        tx, ty, tz = ST_TILE
        return _cdiv(p["nx"], tx) * _cdiv(p["ny"], ty) * _cdiv(p["nz"], tz)
    if kind == "MM":
        return (p["M"] // MM_TILE[0]) * (p["N"] // MM_TILE[1])
    if kind == "MRIQ":
        return _cdiv(p["num_x"], MRIQ_PER_BLOCK)
    if kind == "BS":
        return _cdiv(p["n"], BS_PER_BLOCK)
    if kind == "TEA":
        return _cdiv(p["n"], TEA_PER_BLOCK)
    if kind == "MATADD":
        return (p["n"] // 16) * (p["n"] // 16)
    if kind == "SYNTH":
        return _cdiv(p["n"] // 4, THREADS["SYNTH"] * SYNTH_F4_PER_THREAD)
    raise KeyError(kind)


def _u01(rng, n, lo, hi):
    return (lo + (hi - lo) * rng.random(n, dtype=np.float32)).astype(np.float32)


def _bf16_bits(x: np.ndarray) -> np.ndarray:
    """bf16 bit patterns of float32 values by truncation (inputs only need to be valid bf16)."""
    return (x.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)


def gen(kind: str, size="small", seed: int | None = None, mode: str = "random", **over) -> dict:
    """Draw inputs for one kernel instance.

    size: "small" | "paper" | dict of size params.  mode selects special-case inputs used by the
    oracle pins: "int" (small-integer values so fp32 sums are exact), "identity", "linear",
    "shift", "cycle" -- each documented at its kind below.
    """
    if isinstance(size, dict):
        p = dict(size)
    else:
        p = dict((PAPER if size == "paper" else SMALL)[kind])
    p.update(over)
    if seed is None:
        seed = KIND_SEED[kind]
    rng = np.random.default_rng(seed)
    d: dict = {"kind": kind, "params": p, "seed": seed, "mode": mode}

    if kind == "PC":
        n = p["n_nodes"]
        if mode == "cycle":          # next[i] = i+1 mod N: closed form out = start + H mod N
            nxt = ((np.arange(n, dtype=np.int64) + 1) % n).astype(np.int32)
        else:                        # one random N-cycle (Sattolo-equivalent): visit order perm
            perm = rng.permutation(n).astype(np.int64)
            nxt = np.empty(n, dtype=np.int32)
            nxt[perm] = np.roll(perm, -1).astype(np.int32)
        d["next"] = nxt
    elif kind == "SAD":
        w, h = p["width"], p["height"]
        cur = rng.integers(0, 256, size=(h, w), dtype=np.uint8)
        if mode == "shift":          # ref(x+u, y+v) = cur(x, y): SAD = 0 at offset (u, v) inside
            u, v = over.get("u", 3), over.get("v", -5)
            ref = np.roll(np.roll(cur, v, axis=0), u, axis=1).copy()
        elif mode == "identical":
            ref = cur.copy()
        else:
            ref = rng.integers(0, 256, size=(h, w), dtype=np.uint8)
        d["cur"], d["ref"] = cur, ref
    elif kind == "SPMV":
        nr, nc = p["n_rows"], p["n_cols"]
        lo, hi = p["nnz_min"], p["nnz_max"]
        if mode == "identity":
            assert nr <= nc
            lens = np.ones(nr, dtype=np.int64)
            cols = np.arange(nr, dtype=np.int32)
            vals = np.ones(nr, dtype=np.float32)
        else:
            lens = rng.integers(lo, hi + 1, size=nr)
            # hi sorted distinct columns per row: sorted draws in [0, nc-hi) plus 0..hi-1
            cand = np.sort(rng.integers(0, nc - hi, size=(nr, hi)), axis=1) + np.arange(hi)
            mask = np.arange(hi)[None, :] < lens[:, None]
            cols = cand[mask].astype(np.int32)
            if mode == "int":
                vals = rng.integers(-4, 5, size=cols.size).astype(np.float32)
            else:
                vals = _u01(rng, cols.size, -1.0, 1.0)
        rowptr = np.zeros(nr + 1, dtype=np.int32)
        rowptr[1:] = np.cumsum(lens)
        if mode == "int":
            x = rng.integers(-4, 5, size=nc).astype(np.float32)
        else:
            x = _u01(rng, nc, -1.0, 1.0)
        d.update(rowptr=rowptr, cols=cols, vals=vals, x=x)
    elif kind == "ST":
        nx, ny, nz = p["nx"], p["ny"], p["nz"]
        if mode == "linear":         # a*x + b*y + c*z + e: discrete Laplacian is exactly 0 inside
            z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
            a = (3 * x - 2 * y + 5 * z + 7).astype(np.float32)
        elif mode == "int":
            a = rng.integers(-64, 65, size=(nz, ny, nx)).astype(np.float32)
        else:
            a = _u01(rng, nz * ny * nx, -1.0, 1.0).reshape(nz, ny, nx)
        d["inp"] = np.ascontiguousarray(a)
    elif kind == "MM":
        M, N, K = p["M"], p["N"], p["K"]
        if mode == "int":            # integers in [-8, 8] are exact in bf16; every partial sum exact
            A = rng.integers(-8, 9, size=(M, K)).astype(np.float32)
            Bt = rng.integers(-8, 9, size=(N, K)).astype(np.float32)
        else:
            A = _u01(rng, M * K, -1.0, 1.0).reshape(M, K)
            Bt = _u01(rng, N * K, -1.0, 1.0).reshape(N, K)
        d["A"], d["Bt"] = _bf16_bits(A), _bf16_bits(Bt)   # bf16 bits; B stored K-major (N x K)
    elif kind == "MRIQ":
        nx_, nk = p["num_x"], p["num_k"]
        d["x"] = _u01(rng, nx_, -0.5, 0.5)
        d["y"] = _u01(rng, nx_, -0.5, 0.5)
        d["z"] = _u01(rng, nx_, -0.5, 0.5)
        if mode == "zero_k":        # k = 0: Qr = sum phiMag, Qi = 0
            d["kx"] = np.zeros(nk, np.float32); d["ky"] = np.zeros(nk, np.float32)
            d["kz"] = np.zeros(nk, np.float32)
        else:
            d["kx"] = _u01(rng, nk, -32.0, 32.0)
            d["ky"] = _u01(rng, nk, -32.0, 32.0)
            d["kz"] = _u01(rng, nk, -32.0, 32.0)
        d["phimag"] = _u01(rng, nk, 0.0, 2.0)
    elif kind == "BS":
        n = p["n"]
        d["S"] = _u01(rng, n, 5.0, 30.0)
        d["X"] = _u01(rng, n, 1.0, 100.0)
        d["T"] = _u01(rng, n, 0.25, 10.0)
        p.setdefault("R", 0.02)
        p.setdefault("V", 0.30)
    elif kind == "TEA":
        n = p["n"]
        d["v"] = rng.integers(0, 1 << 32, size=2 * n, dtype=np.uint64).astype(np.uint32)
        d["key"] = rng.integers(0, 1 << 32, size=4, dtype=np.uint64).astype(np.uint32)
    elif kind == "MATADD":
        n = p["n"]
        d["A"] = _u01(rng, n * n, -1.0, 1.0).reshape(n, n)
        d["B"] = _u01(rng, n * n, -1.0, 1.0).reshape(n, n)
    elif kind == "SYNTH":
        d["x"] = _u01(rng, p["n"], -1.0, 1.0)
        p.setdefault("a", 0.999)
        p.setdefault("b", 0.001)
    else:
        raise KeyError(kind)

    d["grid_blocks"] = grid_blocks(kind, p)
    d["threads"] = THREADS[kind]
    return d


# ---------------------------------------------------------------------------------------------
# Workload mixes (PAPER.md tb:workloads) and Poisson arrivals
# ---------------------------------------------------------------------------------------------
MIXES = {
    "CI": ["BS", "MM", "TEA", "MRIQ"],
    "MI": ["PC", "SPMV", "ST", "SAD"],
    "MIX": ["PC", "BS", "TEA", "SAD"],
    "ALL": ["PC", "SPMV", "ST", "BS", "MM", "TEA", "MRIQ", "SAD"],
}


def queue(mix: str = "ALL", n_kernels: int = 8, seed: int = 42, order: str = "round_robin",
          lam: float = 1e6) -> list[dict]:
    """A kernel submission queue: list of {kind, arrival} in arrival order.

    order="round_robin": n_kernels // len(mix) instances of each member kernel in mix order
    (config C2: one or four instances of each kernel of ALL).
    order="uniform": n_kernels drawn uniformly from the mix (config C4, seed 42).
    Arrivals: each application is a Poisson stream with the same rate lam;
    the merged arrival times are returned (lam large => effectively all pending at t~0).
    """
    rng = np.random.default_rng(seed)
    members = MIXES[mix] if mix in MIXES else list(mix)
    if order == "round_robin":
        # deterministic arrival order: evenly spaced at 1/lam
        return [{"kind": members[i % len(members)], "arrival": i / lam} for i in range(n_kernels)]
    kinds = [members[int(i)] for i in rng.integers(0, len(members), size=n_kernels)]
    # per-application Poisson streams (exponential inter-arrival times, rate lam each)
    t_app = {k: 0.0 for k in members}
    out = []
    for k in kinds:
        t_app[k] += float(rng.exponential(1.0 / lam))
        out.append({"kind": k, "arrival": t_app[k]})
    out.sort(key=lambda e: e["arrival"])
    return out


def multi_user_queue(n_kernels: int = 10000, n_users: int = 16, seed: int = 7,
                     lam: float = 1e6) -> list[dict]:
    """Config C5: n_users users, each a Poisson stream from one mix (CI/MI/MIX/ALL round-robin
    over users, seed 7+u), merged by arrival time, truncated to n_kernels."""
    names = ["CI", "MI", "MIX", "ALL"]
    per = -(-n_kernels // n_users)
    allq = []
    for u in range(n_users):
        q = queue(names[u % 4], per, seed=seed + u, order="uniform", lam=lam)
        for e in q:
            e["user"] = u
        allq.extend(q)
    allq.sort(key=lambda e: (e["arrival"], e["user"]))
    return allq[:n_kernels]

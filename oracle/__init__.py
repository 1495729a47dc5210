"""CPU oracle for the Kernelet hot path -- TEST INFRASTRUCTURE, NOT THE PRODUCT.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference) may
import this package.  It shares no code with the CUDA path (paper_1303_5164_b200/): the
arithmetic lives in plain C (oracle/kernels.c, oracle/model.c, built by build() below into
oracle/liboracle.so with -O2 -fno-fast-math -ffp-contract=off) and the scheduling control
logic (candidate space, pruning, FindCoSchedule, Alg.1, brute force) is plain Python here.
The only module both sides use is kl_inputs (seeded input generators, no method arithmetic).

Citations: P:n = /root/reference/PAPER.md line n; readings R1..R25 = SURVEY.md §8(c), restated
in DESIGN.md §3.  Parity-unpinned parts: the model-vs-hardware error and the calibrated
constants (L0, B, a0, b0, alpha_p, alpha_m on B200) -- see DESIGN.md §3.
"""
from __future__ import annotations

import ctypes as C
import itertools
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, f) for f in ("kernels.c", "model.c", "model3.c")]


def build(force: bool = False) -> str:
    """Compile the C oracle (plain gcc, strict IEEE evaluation order)."""
    newest = max(os.path.getmtime(s) for s in _SRC + [os.path.join(_HERE, "oracle.h")])
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-std=c11", "-fPIC",
               "-shared", "-o", _SO] + _SRC + ["-lm"]
        subprocess.run(cmd, check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_SO)
        _declare(_lib)
    return _lib


class SmCfg(C.Structure):
    _fields_ = [("L0", C.c_double), ("B", C.c_double), ("a0", C.c_double), ("b0", C.c_double),
                ("W", C.c_int), ("latency_mode", C.c_int), ("pir_mode", C.c_int),
                ("const_q", C.c_double)]


class KModel(C.Structure):
    _fields_ = [("rm", C.c_double), ("r", C.c_double), ("ipb", C.c_double), ("wpb", C.c_int),
                ("pi", C.c_double), ("pipe", C.c_int)]


class KModel3(C.Structure):
    """f1 three-state kind descriptor (oracle/model3.c, reading R27)."""
    _fields_ = [("rm", C.c_double), ("r", C.c_double), ("uc", C.c_double), ("ru", C.c_double),
                ("ipb", C.c_double), ("wpb", C.c_int), ("pi", C.c_double), ("pipe", C.c_int), ("g", C.c_int)]


class Pred(C.Structure):
    _fields_ = [("ipc1", C.c_double), ("ipc2", C.c_double), ("c", C.c_double),
                ("solo1", C.c_double), ("solo2", C.c_double), ("cp", C.c_double),
                ("dT", C.c_double), ("status", C.c_int)]


class SmRes(C.Structure):
    _fields_ = [("max_warps", C.c_int), ("max_blocks", C.c_int), ("max_regs", C.c_int),
                ("max_smem", C.c_int), ("max_tmem_cols", C.c_int), ("reg_unit", C.c_int)]


class KRes(C.Structure):
    _fields_ = [("wpb", C.c_int), ("regs", C.c_int), ("smem", C.c_int), ("tmem", C.c_int)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)


def _declare(L):
    L.or_latency.restype = C.c_double
    L.or_latency.argtypes = [C.POINTER(SmCfg), C.c_double, C.c_int]
    L.or_row.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _D]
    L.or_build_homog.argtypes = [C.POINTER(KModel), C.c_int, C.POINTER(SmCfg), _D, _D]
    L.or_build_joint.argtypes = [C.POINTER(KModel), C.c_int, C.POINTER(KModel), C.c_int,
                                 C.POINTER(SmCfg), _D, _D]
    L.or_stationary.argtypes = [C.c_int, _D, _D]
    L.or_ipc_homog.restype = C.c_double
    L.or_ipc_homog.argtypes = [C.c_int, _D]
    L.or_ipc_homog_r.restype = C.c_double
    L.or_ipc_homog_r.argtypes = [C.c_int, _D, _D]
    L.or_ipc_joint.argtypes = [C.c_int, C.c_int, _D, _D, _D, _D, _D]
    L.or_cp.restype = C.c_double
    L.or_cp.argtypes = [C.c_int, _D, _D]
    L.or_predict.argtypes = [C.POINTER(KModel), C.c_int, C.c_int, C.POINTER(KModel), C.c_int,
                             C.c_int, C.c_int, C.POINTER(SmCfg), C.POINTER(Pred)]
    L.or_solo_ipc.restype = C.c_double
    L.or_solo_ipc.argtypes = [C.POINTER(KModel), C.c_int, C.c_int, C.POINTER(SmCfg),
                              C.POINTER(C.c_int)]
    L.or3_nstates.argtypes = [C.c_int]
    L.or3_row.argtypes = [C.POINTER(KModel3), C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, _D]
    L.or3_build.argtypes = [C.POINTER(KModel3), C.c_int, C.POINTER(KModel3), C.c_int, C.POINTER(SmCfg), _D, _D]
    L.or3_ipc.argtypes = [C.c_int, C.c_int, C.c_int, _D, _D, _D, _D]
    L.or3_ipc_g.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _D, _D, _D, _D]
    L.or3_solo_ipc.restype = C.c_double
    L.or3_solo_ipc.argtypes = [C.POINTER(KModel3), C.c_int, C.c_int, C.POINTER(SmCfg), C.POINTER(C.c_int)]
    L.or3_predict.argtypes = [C.POINTER(KModel3), C.c_int, C.c_int, C.POINTER(KModel3), C.c_int, C.c_int,
                              C.c_int, C.POINTER(SmCfg), C.POINTER(Pred)]
    L.or_fits.argtypes = [C.POINTER(SmRes), C.POINTER(KRes), C.c_int, C.POINTER(KRes), C.c_int]
    L.or_max_blocks.argtypes = [C.POINTER(SmRes), C.POINTER(KRes)]
    L.or_pruned.argtypes = [C.c_double] * 6
    L.or_cnd.restype = C.c_double
    L.or_cnd.argtypes = [C.c_double]
    for name in ("or_pc", "or_sad", "or_spmv", "or_stencil", "or_mm", "or_mriq", "or_bs",
                 "or_tea", "or_tea_decrypt", "or_matadd", "or_synth"):
        getattr(L, name).restype = None


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _dptr(a):
    return a.ctypes.data_as(_D)


# =============================================================================================
# O1: kernels (definitions in oracle/kernels.c).  Each takes a kl_inputs.gen() dict and an
# optional array of flat output indices; returns a dict of numpy outputs.
# =============================================================================================
def run_kernel(d: dict, idx=None, **kw) -> dict:
    L = lib()
    k = d["kind"]
    p = d["params"]
    ix = None if idx is None else np.ascontiguousarray(idx, dtype=np.int64)
    nix = 0 if ix is None else ix.size
    ixp = _ptr(ix)

    def n_out(n_all):
        return n_all if ix is None else nix

    if k == "PC":
        n = n_out(p["n_threads"])
        o_p = np.empty(n, np.int32)
        o_a = np.empty(n, np.uint32)
        L.or_pc(_ptr(d["next"]), C.c_uint32(p["n_nodes"]), C.c_uint32(p["hops"]),
                C.c_uint32(p["n_threads"]), ixp, C.c_size_t(nix), _ptr(o_p), _ptr(o_a))
        return {"out": o_p, "acc": o_a}
    if k == "SAD":
        w, h = p["width"], p["height"]
        n = n_out((w // 16) * (h // 16) * 1089)
        o = np.empty(n, np.uint16)
        L.or_sad(_ptr(d["cur"]), _ptr(d["ref"]), C.c_int(w), C.c_int(h), ixp, C.c_size_t(nix),
                 _ptr(o))
        return {"sad": o}
    if k == "SPMV":
        n = n_out(p["n_rows"])
        y = np.empty(n, np.float32)
        a = np.empty(n, np.float64)
        L.or_spmv(_ptr(d["rowptr"]), _ptr(d["cols"]), _ptr(d["vals"]), _ptr(d["x"]),
                  C.c_int(p["n_rows"]), ixp, C.c_size_t(nix), _ptr(y), _ptr(a))
        return {"y": y, "scale": a}
    if k == "ST":
        nx, ny, nz = p["nx"], p["ny"], p["nz"]
        c0 = kw.get("c0", p.get("c0", 1.0 / 6.0))
        c1 = kw.get("c1", p.get("c1", 1.0 / 36.0))
        n = n_out(nx * ny * nz)
        o = np.empty(n, np.float32)
        a = np.empty(n, np.float64)
        L.or_stencil(_ptr(d["inp"]), C.c_int(nx), C.c_int(ny), C.c_int(nz),
                     C.c_float(np.float32(c0)), C.c_float(np.float32(c1)), ixp, C.c_size_t(nix),
                     _ptr(o), _ptr(a))
        return {"out": o, "scale": a}
    if k == "MM":
        M, N, K = p["M"], p["N"], p["K"]
        n = n_out(M * N)
        o = np.empty(n, np.float32)
        a = np.empty(n, np.float64)
        L.or_mm(_ptr(d["A"]), _ptr(d["Bt"]), C.c_int(M), C.c_int(N), C.c_int(K), ixp,
                C.c_size_t(nix), _ptr(o), _ptr(a))
        return {"C": o, "scale": a}
    if k == "MRIQ":
        n = n_out(p["num_x"])
        qr = np.empty(n, np.float32)
        qi = np.empty(n, np.float32)
        a = np.empty(n, np.float64)
        L.or_mriq(_ptr(d["x"]), _ptr(d["y"]), _ptr(d["z"]), C.c_int(p["num_x"]), _ptr(d["kx"]),
                  _ptr(d["ky"]), _ptr(d["kz"]), _ptr(d["phimag"]), C.c_int(p["num_k"]), ixp,
                  C.c_size_t(nix), _ptr(qr), _ptr(qi), _ptr(a))
        return {"qr": qr, "qi": qi, "scale": a}
    if k == "BS":
        n = n_out(p["n"])
        call = np.empty(n, np.float32)
        put = np.empty(n, np.float32)
        mag = np.empty(n, np.float64)
        L.or_bs(_ptr(d["S"]), _ptr(d["X"]), _ptr(d["T"]), C.c_size_t(p["n"]),
                C.c_double(p["R"]), C.c_double(p["V"]), ixp, C.c_size_t(nix), _ptr(call),
                _ptr(put), _ptr(mag))
        return {"call": call, "put": put, "scale": mag}
    if k == "TEA":
        n = n_out(p["n"])
        o = np.empty(2 * n, np.uint32)
        L.or_tea(_ptr(d["v"]), C.c_size_t(p["n"]), _ptr(d["key"]), ixp, C.c_size_t(nix), _ptr(o))
        return {"out": o}
    if k == "MATADD":
        n = p["n"]
        o = np.empty((n, n), np.float32)
        L.or_matadd(_ptr(d["A"]), _ptr(d["B"]), C.c_int(n), _ptr(o))
        return {"C": o}
    if k == "SYNTH":
        n = n_out(p["n"])
        o = np.empty(n, np.float32)
        L.or_synth(_ptr(d["x"]), C.c_size_t(p["n"]), C.c_int(p["fmas"]),
                   C.c_float(np.float32(p["a"])), C.c_float(np.float32(p["b"])), ixp,
                   C.c_size_t(nix), _ptr(o))
        return {"y": o}
    raise KeyError(k)


def tea_decrypt(v: np.ndarray, key: np.ndarray) -> np.ndarray:
    out = np.empty_like(v)
    lib().or_tea_decrypt(_ptr(v), C.c_size_t(v.size // 2), _ptr(key), _ptr(out))
    return out


def cnd(d: float) -> float:
    return lib().or_cnd(d)


# =============================================================================================
# O2: Markov model (oracle/model.c).  Python only marshals arrays.
# =============================================================================================
def smcfg(L0=800.0, B=1.0, a0=0.0, b0=0.0, W=16, latency_mode=0, pir_mode=0, const_q=0.0):
    return SmCfg(L0, B, a0, b0, W, latency_mode, pir_mode, const_q)


def kmodel(rm, r=1.0, ipb=1000.0, wpb=4, pi=1.0, pipe=0):
    return KModel(rm, r, ipb, wpb, pi, pipe)


def latency(cfg, n, idle=0):
    return lib().or_latency(C.byref(cfg), n, idle)


def row(w, i, p_ir, rm):
    r = np.zeros(w + 1)
    lib().or_row(w, i, p_ir, rm, _dptr(r))
    return r


def build_homog(k, w, cfg):
    P = np.zeros((w + 1, w + 1))
    R = np.zeros(w + 1)
    rc = lib().or_build_homog(C.byref(k), w, C.byref(cfg), _dptr(P), _dptr(R))
    if rc:
        raise ValueError("latency guard L > W failed (R22)")
    return P, R


def build_joint(k1, w1, k2, w2, cfg):
    S = (w1 + 1) * (w2 + 1)
    P = np.zeros((S, S))
    R = np.zeros(S)
    rc = lib().or_build_joint(C.byref(k1), w1, C.byref(k2), w2, C.byref(cfg), _dptr(P), _dptr(R))
    if rc:
        raise ValueError("latency guard L > W failed (R22)")
    return P, R


def stationary(P):
    P = np.ascontiguousarray(P, dtype=np.float64)
    pi = np.zeros(P.shape[0])
    if lib().or_stationary(P.shape[0], _dptr(P), _dptr(pi)):
        raise ValueError("singular chain")
    return pi


def ipc_homog(w, pi, R=None):
    if R is None:
        return lib().or_ipc_homog(w, _dptr(np.ascontiguousarray(pi)))
    return lib().or_ipc_homog_r(w, _dptr(np.ascontiguousarray(pi)), _dptr(np.ascontiguousarray(R)))


def ipc_joint(w1, w2, pi, R):
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    lib().or_ipc_joint(w1, w2, _dptr(np.ascontiguousarray(pi)), _dptr(np.ascontiguousarray(R)),
                       C.byref(a), C.byref(b), C.byref(c))
    return a.value, b.value, c.value


def cp(cipc, ipc):
    ci = np.ascontiguousarray(cipc, dtype=np.float64)
    ip = np.ascontiguousarray(ipc, dtype=np.float64)
    return lib().or_cp(len(ci), _dptr(ci), _dptr(ip))


def predict(k1, b1, b1max, k2, b2, b2max, nsched, cfg) -> Pred:
    out = Pred()
    lib().or_predict(C.byref(k1), b1, b1max, C.byref(k2), b2, b2max, nsched, C.byref(cfg),
                     C.byref(out))
    return out


# ---- f1: three-state model (oracle/model3.c, reading R27) ---------------------
def kmodel3(rm, r=1.0, uc=0.0, ru=None, ipb=1000.0, wpb=4, pi=1.0, pipe=0, g=1):
    return KModel3(rm, r, uc, r if ru is None else ru, ipb, wpb, pi, pipe, g)


def nstates3(w):
    return lib().or3_nstates(w)


def row3(k, w, c, u, pc, pu):
    r = np.zeros(nstates3(w))
    lib().or3_row(C.byref(k), w, c, u, pc, pu, _dptr(r))
    return r


def build3(k1, w1, cfg, k2=None, w2=0):
    S = nstates3(w1) * (nstates3(w2) if k2 is not None else 1)
    P = np.zeros((S, S))
    R = np.zeros(S)
    rc = lib().or3_build(C.byref(k1), w1, C.byref(k2) if k2 is not None else None, w2 if k2 is not None else 0,
                         C.byref(cfg), _dptr(P), _dptr(R))
    if rc:
        raise ValueError("latency guard L > W failed (R22)")
    return P, R


def ipc3(w1, pi, R, w2=None, g1=1, g2=1):
    a, b = C.c_double(), C.c_double()
    lib().or3_ipc_g(w1, g1, w2 or 0, g2, 1 if w2 is not None else 0, _dptr(np.ascontiguousarray(pi)),
                    _dptr(np.ascontiguousarray(R)), C.byref(a), C.byref(b))
    return (a.value, b.value) if w2 is not None else a.value


def states3(w):
    """(c, u) of every state index of one kernel (model3.c idx3 order)."""
    return [(c, u) for c in range(w + 1) for u in range(w - c + 1)]


def predict3(k1, b1, b1max, k2, b2, b2max, nsched, cfg) -> Pred:
    out = Pred()
    lib().or3_predict(C.byref(k1), b1, b1max, C.byref(k2), b2, b2max, nsched, C.byref(cfg), C.byref(out))
    return out


def solo_ipc3(k, b, nsched, cfg):
    st = C.c_int()
    v = lib().or3_solo_ipc(C.byref(k), b, nsched, C.byref(cfg), C.byref(st))
    if st.value:
        raise ValueError(f"solo three-state model failed ({st.value})")
    return v


def solo_ipc(k, b, nsched, cfg):
    st = C.c_int()
    v = lib().or_solo_ipc(C.byref(k), b, nsched, C.byref(cfg), C.byref(st))
    return v, st.value


# =============================================================================================
# O3: occupancy, pruning (oracle/model.c)
# =============================================================================================
B200_SM = dict(max_warps=64, max_blocks=32, max_regs=65536, max_smem=233472, max_tmem_cols=512,
               reg_unit=256)
FERMI_SM = dict(max_warps=48, max_blocks=8, max_regs=32768, max_smem=49152 + 8 * 1024,
                max_tmem_cols=0, reg_unit=64)
KEPLER_SM = dict(max_warps=64, max_blocks=16, max_regs=65536, max_smem=49152 + 16 * 1024,
                 max_tmem_cols=0, reg_unit=256)


def fits(sm: dict, r1: dict, b1: int, r2: dict | None = None, b2: int = 0) -> int:
    s = SmRes(**sm)
    k1 = KRes(r1["wpb"], r1["regs"], r1["smem"], r1.get("tmem", 0))
    k2 = KRes(r2["wpb"], r2["regs"], r2["smem"], r2.get("tmem", 0)) if r2 else None
    return lib().or_fits(C.byref(s), C.byref(k1), b1, C.byref(k2) if k2 else None, b2)


def max_blocks(sm: dict, r: dict) -> int:
    s = SmRes(**sm)
    k = KRes(r["wpb"], r["regs"], r["smem"], r.get("tmem", 0))
    return lib().or_max_blocks(C.byref(s), C.byref(k))


def pruned(pur1, mur1, pur2, mur2, ap, am) -> bool:
    return bool(lib().or_pruned(pur1, mur1, pur2, mur2, ap, am))


# =============================================================================================
# Scheduling control logic: candidate space, FindCoSchedule, Alg.1.
# =============================================================================================
BAND = 1e-12


def _band(x, y):
    return BAND * max(1.0, abs(x), abs(y))


def levels(prof: dict, nsched: int = 4, mode: str = "all") -> list[int]:
    """Candidate blocks-per-SM levels of a kind (a5): b in 1..b_max with b*wpb divisible by the
    scheduler count (whole warps per virtual SM, R14); mode "4" keeps the four levels
    {1/4, 1/2, 3/4, 1} * b_max rounded up to such a b (config C2)."""
    bmax, wpb = prof["bmax"], prof["wpb"]
    ok = [b for b in range(1, bmax + 1) if (b * wpb) % nsched == 0]
    if mode == "all":
        return ok
    out = []
    for q in (1, 2, 3, 4):
        t = -(-q * bmax // 4)
        c = [b for b in ok if b >= t]
        if c and c[0] not in out:
            out.append(c[0])
    return out


def solo_b(prof: dict, nsched: int = 4) -> int:
    """Solo maximum occupancy level b_max (the IPC_i of Eq.1 is the solo IPC at b_max); 0 if no
    occupancy gives whole warps per virtual SM."""
    lv = levels(prof, nsched, "all")
    return lv[-1] if lv else 0


def maximal_splits(sm: dict, p1: dict, p2: dict, nsched=4, mode="all") -> list[tuple[int, int]]:
    """Feasible (b1, b2) co-residencies that cannot grow either kernel (R7), (b1, b2) order."""
    l1, l2 = levels(p1, nsched, mode), levels(p2, nsched, mode)
    feas = [(a, b) for a in l1 for b in l2 if fits(sm, p1, a, p2, b) == 0]
    fs = set(feas)
    out = []
    for a, b in feas:
        dom = any((x, y) in fs and (x, y) != (a, b) and x >= a and y >= b for x in l1 for y in l2)
        if not dom:
            out.append((a, b))
    return sorted(out)


def kmodel_of(prof: dict) -> KModel:
    return KModel(prof["rm"], prof["r"], prof["ipb"], prof["wpb"], prof.get("ipc_max", 1.0) or 1.0,
                  int(prof.get("pipe", 0)))


def kmodel3_of(prof: dict, states: int = 3, granularity: int = 0, nsched: int = 4) -> KModel3:
    """f1 descriptor: three-state only when configured and the kind has uncoalesced accesses
    (uc > 0); block granularity (R13) models units of wpb/nsched warps when wpb divides evenly."""
    uc = float(prof.get("uc", 0.0) or 0.0) if states == 3 else 0.0
    r = prof["r"]
    ru = float(prof.get("ru", 0.0) or 0.0) or r
    wpb = prof["wpb"]
    g = wpb // nsched if (granularity == 1 and wpb % nsched == 0 and wpb >= nsched) else 1
    return KModel3(prof["rm"], r, uc, ru, prof["ipb"], wpb, prof.get("ipc_max", 1.0) or 1.0,
                   int(prof.get("pipe", 0)), g)


def predict_cfg(p1, b1, p2, b2, cfg, nsched=4, states=2, granularity=0) -> Pred:
    """The model prediction the runtime's configuration selects: two-state warp model
    (oracle/model.c) by default, else the f1 chain (oracle/model3.c)."""
    if states == 2 and granularity == 0:
        return predict(kmodel_of(p1), b1, solo_b(p1, nsched), kmodel_of(p2), b2, solo_b(p2, nsched), nsched, cfg)
    return predict3(kmodel3_of(p1, states, granularity, nsched), b1, solo_b(p1, nsched),
                    kmodel3_of(p2, states, granularity, nsched), b2, solo_b(p2, nsched), nsched, cfg)


def pairs_of(pending: list[dict], distinct_kinds: bool = False) -> list[tuple[int, int]]:
    """Candidate pairs over pending instances in arrival order, one pair per
    unordered kind pair (earliest instances), same-kind pairs included when two instances of a
    kind are pending -- unless `distinct_kinds` (reading R31b: with saturation b_max a same-kind
    pair is the kind at b1 + b2 >= b_sat blocks, no faster than solo).  Returns index pairs into
    `pending`."""
    reps, seen_k = [], {}
    for i, e in enumerate(pending):
        c = seen_k.get(e["kind"], 0)
        if c < 2:
            reps.append(i)
            seen_k[e["kind"]] = c + 1
    out, seen = [], set()
    for a, b in itertools.combinations(reps, 2):
        key = tuple(sorted((pending[a]["kind"], pending[b]["kind"])))
        if key in seen or (distinct_kinds and key[0] == key[1]):
            continue
        seen.add(key)
        out.append((a, b))
    return out


def prune(pending, pairs, profs, ap, am):
    """Pruning with AND semantics (R9); if everything is pruned, halve both
    thresholds (R10) at most 8 times, then disable pruning (R24)."""
    for it in range(10):
        if it == 9:
            ap = am = 0.0
        keep = [pq for pq in pairs
                if not pruned(profs[pending[pq[0]]["kind"]]["pur"],
                              profs[pending[pq[0]]["kind"]]["mur"],
                              profs[pending[pq[1]]["kind"]]["pur"],
                              profs[pending[pq[1]]["kind"]]["mur"], ap, am)]
        if keep or not pairs:
            return keep, (ap, am)
        ap, am = ap / 2, am / 2
    return pairs, (0.0, 0.0)


def _better_split(a, b, rule=0):
    """a9: argmin dT; ties: larger C, then more warps, then smaller b1.  rule 1 (ablation):
    highest CP first, then the same order."""
    if rule == 1:
        t = _band(a["cp"], b["cp"])
        if a["cp"] > b["cp"] + t:
            return True
        if a["cp"] < b["cp"] - t:
            return False
    # dT ties relative to the Eq.8 terms (R8): dT is a difference of per-wave times, so its
    # rounding noise scales with them
    t = 1e-9 * max(a["dT_scale"], b["dT_scale"])
    if a["dT"] < b["dT"] - t:
        return True
    if a["dT"] > b["dT"] + t:
        return False
    t = _band(a["c"], b["c"])
    if a["c"] > b["c"] + t:
        return True
    if a["c"] < b["c"] - t:
        return False
    if a["warps"] != b["warps"]:
        return a["warps"] > b["warps"]
    return a["b1"] < b["b1"]


def find_co_schedule(pending: list[dict], profs: dict, cfg: SmCfg, sm=B200_SM, nsched=4,
                     ap=0.4, am=0.1, mode="all", n_sm=148, cache=None, cp_min=0.0, split_rule=0,
                     states=2, granularity=0, distinct_kinds=False) -> dict:
    """Proc. FindCoSchedule: candidates -> prune -> model CP -> argmax.

    Per surviving pair the slice ratio is the argmin of dT (Eq.8) over maximal splits; across
    pairs the max CP wins (ties: earliest pair).  Best CP <= 0 (R25) or < 2 candidates: the
    oldest pending kernel runs solo at b_max.  Slice sizes: size_i = m * b_i * n_sm with the
    common m = max(m_min) of the p% rule (a9)."""
    pairs = pairs_of(pending, distinct_kinds)
    pairs, alphas = prune(pending, pairs, profs, ap, am)
    best = None
    evaluated = []
    for (ia, ib) in pairs:
        p1, p2 = profs[pending[ia]["kind"]], profs[pending[ib]["kind"]]
        bestsplit = None
        for (b1, b2) in maximal_splits(sm, p1, p2, nsched, mode):
            key = (pending[ia]["kind"], pending[ib]["kind"], b1, b2)
            if cache is not None and key in cache:
                pr = cache[key]
            else:
                r = predict_cfg(p1, b1, p2, b2, cfg, nsched, states, granularity)
                pr = dict(ipc1=r.ipc1, ipc2=r.ipc2, c=r.c, solo1=r.solo1, solo2=r.solo2,
                          cp=r.cp, dT=r.dT, status=r.status)
                if cache is not None:
                    cache[key] = pr
            cand = dict(pr, b1=b1, b2=b2, warps=b1 * p1["wpb"] + b2 * p2["wpb"], ia=ia, ib=ib)
            cand["dT_scale"] = (max(p1["ipb"] * b1 / pr["ipc1"], p2["ipb"] * b2 / pr["ipc2"])
                                if pr["status"] == 0 else 0.0)
            evaluated.append(cand)
            if pr["status"] != 0:
                continue
            if bestsplit is None or _better_split(cand, bestsplit, split_rule):
                bestsplit = cand
        if bestsplit is None:
            continue
        if best is None or bestsplit["cp"] > best["cp"] + _band(bestsplit["cp"], best["cp"]):
            best = bestsplit
    if best is None or best["cp"] <= max(BAND, cp_min):
        k = pending[0]
        pr = profs[k["kind"]]
        b = solo_b(pr, nsched)
        return dict(solo=True, ia=0, ib=-1, b1=b, b2=0, cp=0.0, alphas=alphas,
                    evaluated=evaluated, size1=b * n_sm, size2=0)
    p1, p2 = profs[pending[best["ia"]]["kind"]], profs[pending[best["ib"]]["kind"]]
    m = max(p1.get("m_min", 1), p2.get("m_min", 1))
    return dict(best, solo=False, alphas=alphas, evaluated=evaluated,
                size1=m * best["b1"] * n_sm, size2=m * best["b2"] * n_sm)


# ---- predicted makespan (O2 step 11) and brute force -----------------------------------------
def _rate(prof, ipc, n_vsm):
    """Blocks per cycle of a kernel progressing at per-vSM IPC `ipc`."""
    return n_vsm * ipc / prof["ipb"]


def alg1_makespan(queue: list[dict], profs: dict, cfg, sm=B200_SM, nsched=4, ap=0.4, am=0.1,
                  mode="all", n_sm=148, launch_overhead=0.0, decide=None, split_rule=0, cp_min=0.0,
                  distinct_kinds=False):
    """Alg.1 on an all-pending queue, executed in the model: each co-schedule runs
    until either kernel exhausts its blocks (R11), then the scheduler re-plans.  Returns
    (makespan in cycles, trace)."""
    n_vsm = nsched * n_sm
    pend = [dict(e, rem=float(e["blocks"])) for e in queue]
    t, trace, cache = 0.0, [], {}
    while pend:
        dec = decide(pend) if decide else find_co_schedule(pend, profs, cfg, sm, nsched, ap, am,
                                                           mode, n_sm, cache, split_rule=split_rule, cp_min=cp_min,
                                                           distinct_kinds=distinct_kinds)
        if dec["solo"]:
            k = pend[dec["ia"]]
            pr = profs[k["kind"]]
            ipc, _ = solo_ipc(kmodel_of(pr), solo_b(pr, nsched), nsched, cfg)
            dt = k["rem"] / _rate(pr, ipc, n_vsm)
            trace.append(("solo", k["kind"], dt))
            pend.pop(dec["ia"])
        else:
            a, b = pend[dec["ia"]], pend[dec["ib"]]
            ra = _rate(profs[a["kind"]], dec["ipc1"], n_vsm)
            rb = _rate(profs[b["kind"]], dec["ipc2"], n_vsm)
            dt = min(a["rem"] / ra, b["rem"] / rb)
            a["rem"] -= dt * ra
            b["rem"] -= dt * rb
            trace.append(("pair", a["kind"], b["kind"], dec["b1"], dec["b2"], dt))
            pend = [e for e in pend if e["rem"] > 1e-9 * e["blocks"]]
        t += dt + launch_overhead
    return t, trace


def brute_force_makespan(queue, profs, cfg, sm=B200_SM, nsched=4, mode="all", n_sm=148,
                         launch_overhead=0.0):
    """Minimum model makespan over every decision sequence (any pair, any maximal split, or any
    kernel solo) at every completion point -- the optimum of the problem definition
    within the pairwise, fixed-ratio-per-phase plan space.  Tiny queues only."""
    n_vsm = nsched * n_sm
    memo = {}

    def solo_rate(kind):
        pr = profs[kind]
        ipc, _ = solo_ipc(kmodel_of(pr), solo_b(pr, nsched), nsched, cfg)
        return _rate(pr, ipc, n_vsm)

    def rec(state):
        if not state:
            return 0.0
        if state in memo:
            return memo[state]
        best = float("inf")
        items = list(state)
        for i, (kind, rem) in enumerate(items):
            rest = tuple(items[:i] + items[i + 1:])
            best = min(best, rem / solo_rate(kind) + launch_overhead + rec(rest))
        for i, j in itertools.combinations(range(len(items)), 2):
            (ka, ra_), (kb, rb_) = items[i], items[j]
            pa, pb = profs[ka], profs[kb]
            for b1, b2 in maximal_splits(sm, pa, pb, nsched, mode):
                r = predict(kmodel_of(pa), b1, solo_b(pa, nsched), kmodel_of(pb), b2,
                            solo_b(pb, nsched), nsched, cfg)
                if r.status:
                    continue
                va, vb = _rate(pa, r.ipc1, n_vsm), _rate(pb, r.ipc2, n_vsm)
                dt = min(ra_ / va, rb_ / vb)
                na, nb = ra_ - dt * va, rb_ - dt * vb
                rest = [it for k2, it in enumerate(items) if k2 not in (i, j)]
                if na > 1e-9 * ra_:
                    rest.append((ka, round(na, 6)))
                if nb > 1e-9 * rb_:
                    rest.append((kb, round(nb, 6)))
                best = min(best, dt + launch_overhead + rec(tuple(sorted(rest))))
        memo[state] = best
        return best

    st = tuple(sorted((e["kind"], float(e["blocks"])) for e in queue))
    return rec(st)

"""paper_1303_5164_b200 -- B200-native Kernelet hot path (Zhong & He, arXiv:1303.5164).

Thin ctypes binding of the C ABI in include/kl.h (libkl.so, built from csrc/ for sm_100a).
This module only marshals arguments: every step of the hot path -- slicing, the Markov model,
selection, co-scheduled execution -- runs in libkl.so.  PyTorch provides device memory, streams
and process groups.  There is no CPU fallback: importing the package without libkl.so raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

# The runtime drives a pool of 8 launch streams plus control, stop and caller streams; with the
# default 8 hardware work queues, unrelated streams would share a FIFO and falsely serialise
# (e.g. a launch queued behind an arrival clock).  Effective only if set before the process
# creates its CUDA context, so entry points (bench.py, tools, tests) import this package first.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
LIB_PATH = os.environ.get("KL_LIB_PATH") or os.path.join(_HERE, "libkl.so")   # override: A/B builds
SOURCES = ["csrc/kl_runtime.cpp", "csrc/kl_kernels.cu", "csrc/kl_model.cu", "csrc/kl_model3.cu", "csrc/kl_mm.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC,-O2", "-shared", "-cudart", "static"]


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libkl.so in-tree with nvcc for sm_100a (cross-compiles without a GPU)."""
    srcs = [os.path.join(_HERE, s) for s in SOURCES]
    deps = srcs + [os.path.join(_HERE, "csrc", h) for h in ("kl_internal.h", "kl_launcher.cuh", "kl_model_common.cuh")] + [os.path.join(_ROOT, "include", "kl.h")]
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= max(map(os.path.getmtime, deps)):
        return LIB_PATH
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc] + NVCC_FLAGS + ["-o", LIB_PATH + ".tmp"] + srcs
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=_HERE)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


# ---- enums / constants (mirrors include/kl.h) ----------------------------------------------
KL_OK, KL_EINVAL, KL_EINFEASIBLE, KL_ENOMEM, KL_ECUDA, KL_ENCCL, KL_ENUMERIC, KL_EBUSY, KL_ENOTFOUND = range(9)
STATUS_NAMES = ["KL_OK", "KL_EINVAL", "KL_EINFEASIBLE", "KL_ENOMEM", "KL_ECUDA", "KL_ENCCL",
                "KL_ENUMERIC", "KL_EBUSY", "KL_ENOTFOUND"]
KINDS = ["PC", "SAD", "SPMV", "ST", "MM", "MRIQ", "BS", "TEA", "MATADD", "SYNTH"]
KIND_ID = {k: i for i, k in enumerate(KINDS)}
NKINDS = len(KINDS)

_vp = C.c_void_p
ABI_VERSION = 3   # include/kl.h KL_ABI_VERSION


class ArgsPC(C.Structure):
    _fields_ = [("next", _vp), ("out", _vp), ("acc", _vp), ("n_nodes", C.c_uint32),
                ("hops", C.c_uint32), ("n_threads", C.c_uint32)]


class ArgsSAD(C.Structure):
    _fields_ = [("cur", _vp), ("ref", _vp), ("out", _vp), ("width", C.c_int32), ("height", C.c_int32)]


class ArgsSPMV(C.Structure):
    _fields_ = [("rowptr", _vp), ("cols", _vp), ("vals", _vp), ("x", _vp), ("y", _vp), ("n_rows", C.c_int32)]


class ArgsST(C.Structure):
    _fields_ = [("inp", _vp), ("out", _vp), ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("c0", C.c_float), ("c1", C.c_float)]


class ArgsMM(C.Structure):
    _fields_ = [("A", _vp), ("Bt", _vp), ("C", _vp), ("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32)]


class ArgsMRIQ(C.Structure):
    _fields_ = [("x", _vp), ("y", _vp), ("z", _vp), ("kx", _vp), ("ky", _vp), ("kz", _vp),
                ("phimag", _vp), ("qr", _vp), ("qi", _vp), ("num_x", C.c_int32), ("num_k", C.c_int32)]


class ArgsBS(C.Structure):
    _fields_ = [("S", _vp), ("X", _vp), ("T", _vp), ("call", _vp), ("put", _vp), ("n", C.c_int64),
                ("R", C.c_float), ("V", C.c_float)]


class ArgsTEA(C.Structure):
    _fields_ = [("inp", _vp), ("out", _vp), ("n", C.c_int64), ("key", C.c_uint32 * 4)]


class ArgsMATADD(C.Structure):
    _fields_ = [("A", _vp), ("B", _vp), ("C", _vp), ("n", C.c_int32)]


class ArgsSYNTH(C.Structure):
    _fields_ = [("x", _vp), ("y", _vp), ("n", C.c_int64), ("fmas", C.c_int32), ("a", C.c_float), ("b", C.c_float)]


ARGS = [ArgsPC, ArgsSAD, ArgsSPMV, ArgsST, ArgsMM, ArgsMRIQ, ArgsBS, ArgsTEA, ArgsMATADD, ArgsSYNTH]


class Profile(C.Structure):
    _fields_ = [("rm", C.c_double), ("r", C.c_double), ("ipb", C.c_double), ("pur", C.c_double),
                ("mur", C.c_double), ("wpb", C.c_int32), ("regs", C.c_int32), ("smem", C.c_int32),
                ("tmem", C.c_int32), ("bmax", C.c_int32), ("m_min", C.c_int32), ("ipc_max", C.c_double),
                ("pipe", C.c_int32), ("pad", C.c_int32), ("uc", C.c_double), ("ru", C.c_double)]


class Config(C.Structure):
    _fields_ = [("alpha_p", C.c_double), ("alpha_m", C.c_double), ("p_percent", C.c_double),
                ("L0", C.c_double), ("B", C.c_double), ("a0", C.c_double), ("b0", C.c_double),
                ("cp_min", C.c_double), ("n_sched", C.c_int32), ("latency_mode", C.c_int32), ("level_mode", C.c_int32),
                ("split_rule", C.c_int32), ("model_frozen", C.c_int32),
                ("n_sms", C.c_int32), ("chunk", C.c_int32), ("audit", C.c_int32),
                ("retune", C.c_int32), ("model_states", C.c_int32), ("granularity", C.c_int32),
                ("age_limit_us", C.c_int32), ("mc_seed", C.c_int32), ("speculative", C.c_int32), ("max_regs_per_sm", C.c_int32), ("max_smem_per_sm", C.c_int32),
                ("max_warps_per_sm", C.c_int32), ("max_blocks_per_sm", C.c_int32),
                ("mm_stages", C.c_int32), ("critical", C.c_int32),
                ("distinct_kinds", C.c_int32), ("reserved0", C.c_int32),
                ("profiles", C.POINTER(Profile)), ("stream_a", _vp), ("stream_b", _vp),
                ("counters_dev", _vp)]


class KernelDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("grid_blocks", C.c_uint32), ("args", _vp), ("args_bytes", C.c_uint32),
                ("profile", C.POINTER(Profile)), ("tag", C.c_uint64), ("ready_event", _vp), ("ready_flag", _vp)]


class SlicePlan(C.Structure):
    _fields_ = [("slice_blocks", C.c_uint32), ("n_slices", C.c_uint32), ("blocks_per_sm", C.c_uint32),
                ("waves", C.c_uint32)]


class Candidate(C.Structure):
    _fields_ = [("k1", C.c_int32), ("k2", C.c_int32), ("b1", C.c_uint32), ("b2", C.c_uint32)]


class Prediction(C.Structure):
    _fields_ = [("ipc1", C.c_double), ("ipc2", C.c_double), ("c", C.c_double), ("solo1", C.c_double),
                ("solo2", C.c_double), ("cp", C.c_double), ("dT", C.c_double), ("status", C.c_int32),
                ("pad", C.c_int32)]


class CoSchedule(C.Structure):
    _fields_ = [("id1", C.c_uint64), ("id2", C.c_uint64), ("kind1", C.c_int32), ("kind2", C.c_int32),
                ("b1", C.c_uint32), ("b2", C.c_uint32), ("size1", C.c_uint32), ("size2", C.c_uint32),
                ("cp", C.c_double), ("solo", C.c_int32), ("n_candidates", C.c_int32)]


class Counters(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("kernels_done", "blocks_done", "t_start_ns", "t_end_ns",
                                         "checksum", "rank", "world", "phases")]


class Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("decisions", "launches", "stops", "model_batches", "model_candidates",
                                         "device_launches", "decide_ns", "model_ns", "retunes", "topups", "aged", "speculative", "memops")]


class TraceRec(C.Structure):
    _fields_ = [("id", C.c_uint64), ("kind", C.c_int32), ("lane", C.c_int32), ("cap", C.c_uint32),
                ("slice", C.c_uint32), ("start", C.c_uint32), ("end", C.c_uint32), ("executed", C.c_uint32),
                ("admitted", C.c_uint32), ("max_per_sm", C.c_uint32), ("exhausted", C.c_uint32),
                ("t0_ns", C.c_int64), ("t1_ns", C.c_int64), ("phase", C.c_int32),
                ("partner_kind", C.c_int32), ("cp", C.c_double), ("cap_max", C.c_uint32), ("grids", C.c_uint32),
                ("variant", C.c_uint32), ("pad", C.c_uint32)]


ABI_SYMBOLS = ["kl_abi_version", "kl_config_default", "kl_create", "kl_destroy", "kl_last_error",
               "kl_submit", "kl_slice", "kl_predict", "kl_schedule", "kl_sync", "kl_run_plain",
               "kl_get_profile", "kl_set_profile", "kl_reset_model_cache", "kl_reset_counters",
               "kl_trace", "kl_audit", "kl_decide", "kl_struct_sizes", "kl_stats_get", "kl_run_capped", "kl_run_pair", "kl_cache_put", "kl_submit_batch", "kl_delay", "kl_arrival_clock", "kl_wait_flag", "kl_timeline"]
STRUCTS = ["Config", "Profile", "KernelDesc", "SlicePlan", "Candidate", "Prediction", "CoSchedule",
           "Counters", "TraceRec", "Stats", "ArgsPC", "ArgsSAD", "ArgsSPMV", "ArgsST", "ArgsMM", "ArgsMRIQ",
           "ArgsBS", "ArgsTEA", "ArgsMATADD", "ArgsSYNTH"]

_lib = None


def lib() -> C.CDLL:
    """Load libkl.so (raises if it has not been built -- no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    L.kl_abi_version.restype = C.c_int
    if L.kl_abi_version() != ABI_VERSION:   # the structs below mirror include/kl.h of this version
        raise RuntimeError(f"{LIB_PATH} has ABI {L.kl_abi_version()}, the binding expects {ABI_VERSION}: rebuild")
    L.kl_config_default.argtypes = [P(Config)]
    L.kl_create.argtypes = [C.c_int, P(Config), P(_vp)]
    L.kl_destroy.argtypes = [_vp]
    L.kl_last_error.argtypes = [_vp]
    L.kl_last_error.restype = C.c_char_p
    L.kl_submit.argtypes = [_vp, P(KernelDesc), P(C.c_uint64)]
    L.kl_slice.argtypes = [_vp, C.c_uint64, C.c_uint32, C.c_uint32, P(SlicePlan)]
    L.kl_predict.argtypes = [_vp, P(Candidate), C.c_size_t, P(Prediction)]
    L.kl_schedule.argtypes = [_vp, P(CoSchedule)]
    L.kl_decide.argtypes = [_vp, P(CoSchedule)]
    L.kl_sync.argtypes = [_vp, P(Counters)]
    L.kl_run_plain.argtypes = [_vp, P(KernelDesc), _vp, C.c_uint32, C.c_uint32]
    L.kl_get_profile.argtypes = [_vp, C.c_int, P(Profile)]
    L.kl_set_profile.argtypes = [_vp, C.c_int, P(Profile)]
    L.kl_reset_model_cache.argtypes = [_vp]
    L.kl_reset_counters.argtypes = [_vp]
    L.kl_trace.argtypes = [_vp, P(TraceRec), C.c_size_t, P(C.c_size_t)]
    L.kl_audit.argtypes = [_vp, C.c_uint64, P(C.c_uint32), C.c_size_t]
    L.kl_struct_sizes.argtypes = [P(C.c_uint32), C.c_int]
    L.kl_stats_get.argtypes = [_vp, P(Stats)]
    L.kl_run_capped.argtypes = [_vp, P(KernelDesc), C.c_uint32, P(C.c_double)]
    L.kl_delay.argtypes = [_vp, C.c_uint64, _vp]
    L.kl_arrival_clock.argtypes = [_vp, _vp, _vp, _vp, C.c_uint32]
    L.kl_wait_flag.argtypes = [_vp, _vp, _vp]
    L.kl_timeline.argtypes = [_vp, C.c_uint64, _vp, C.c_size_t]
    L.kl_submit_batch.argtypes = [_vp, P(KernelDesc), C.c_size_t, P(C.c_uint64)]
    L.kl_cache_put.argtypes = [_vp, P(Candidate), P(Prediction), C.c_size_t]
    L.kl_run_pair.argtypes = [_vp, P(KernelDesc), C.c_uint32, P(KernelDesc), C.c_uint32, P(TraceRec)]
    for s in ABI_SYMBOLS:
        if s not in ("kl_abi_version", "kl_last_error", "kl_struct_sizes"):
            getattr(L, s).restype = C.c_int
    _lib = L
    return L


class KlError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


def default_config(**kw) -> Config:
    c = Config()
    lib().kl_config_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def profile_from_dict(d: dict) -> Profile:
    p = Profile()
    for name, _ in Profile._fields_:
        if name in d:
            setattr(p, name, d[name])
    return p


class Context:
    """One Kernelet scheduler on one CUDA device (queue -> slicer -> model ->
    scheduler -> dispatch).  `device=-1` creates a host-only context."""

    def __init__(self, device: int = 0, config: Config | None = None, profiles: dict | None = None,
                 streams=None, counters=None, **cfg):
        self._L = lib()
        self.config = config or default_config()
        for k, v in cfg.items():
            setattr(self.config, k, v)
        self._prof_arr = None
        if profiles is not None:
            arr = (Profile * NKINDS)()
            for k, d in profiles.items():
                arr[KIND_ID[k] if isinstance(k, str) else k] = profile_from_dict(d) if isinstance(d, dict) else d
            self._prof_arr = arr
            self.config.profiles = C.cast(arr, C.POINTER(Profile))
        if streams is not None:
            self.config.stream_a = streams[0].cuda_stream if hasattr(streams[0], "cuda_stream") else streams[0]
            self.config.stream_b = streams[1].cuda_stream if hasattr(streams[1], "cuda_stream") else streams[1]
        self.counters = counters
        if counters is not None:
            self.config.counters_dev = counters.data_ptr()
        h = _vp()
        st = self._L.kl_create(device, C.byref(self.config), C.byref(h))
        if st != KL_OK:
            raise KlError(st, f"kl_create(device={device}) failed")
        self._h = h
        self._keep = {}   # args structs kept alive until sync

    # -- helpers --
    def _check(self, st):
        if st != KL_OK:
            raise KlError(st, self._L.kl_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._L.kl_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- ABI calls --
    def submit(self, kind, grid_blocks: int, args, tag: int = 0, profile: Profile | None = None,
               ready_event=None) -> int:
        """Alg.1 l.2-3: add a kernel to R.  `ready_event` (torch.cuda.Event or raw cudaEvent_t)
        is waited on by every launch of the kernel (its inputs have landed)."""
        kid = KIND_ID[kind] if isinstance(kind, str) else int(kind)
        ev = getattr(ready_event, "cuda_event", ready_event) if ready_event is not None else None
        d = KernelDesc(kid, grid_blocks, C.cast(C.pointer(args), _vp), C.sizeof(args),
                       C.pointer(profile) if profile is not None else None, tag, ev)
        out = C.c_uint64()
        self._check(self._L.kl_submit(self._h, C.byref(d), C.byref(out)))
        self._keep[out.value] = args
        return out.value

    def delay(self, stream, ns: int, stamp_ptr: int | None = None) -> None:
        """Arrival clock (kl_delay): sleep `ns` of device time on `stream`, then stamp the release
        time (globaltimer ns) at device address `stamp_ptr`."""
        s = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        self._check(self._L.kl_delay(s, int(ns), stamp_ptr))

    def arrival_clock(self, stream, gaps_ptr: int, stamps_ptr: int, flags_ptr: int, n: int) -> None:
        """kl_arrival_clock: one resident thread releases n arrivals (device pointers gaps/stamps,
        host-mapped flags)."""
        s = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        self._check(self._L.kl_arrival_clock(s, gaps_ptr, stamps_ptr, flags_ptr, n))

    def wait_flag(self, stream, flag_ptr: int | None, stamp_ptr: int | None = None) -> None:
        """kl_wait_flag: gate `stream` on a host-visible flag and/or stamp the device time."""
        s = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        self._check(self._L.kl_wait_flag(s, flag_ptr, stamp_ptr))

    def submit_many(self, items) -> list[int]:
        """items: [(kind, grid_blocks, args, tag, ready_event or None[, ready_flag address])]
        -> ids (one ABI call)."""
        n = len(items)
        arr = (KernelDesc * max(n, 1))()
        addressof, sizeof = C.addressof, C.sizeof
        # field-wise fill (addressof, no pointer objects): ~0.5 us per descriptor instead of ~5 us,
        # which at 32 kernels per bench step was 1.5 % of the step in Python marshalling
        for i, it in enumerate(items):
            kind, grid, args, tag, ev = it[:5]
            d = arr[i]
            d.kind = KIND_ID[kind] if isinstance(kind, str) else int(kind)
            d.grid_blocks = grid
            d.args = addressof(args)
            d.args_bytes = sizeof(args)
            d.tag = tag
            if ev is not None:
                d.ready_event = getattr(ev, "cuda_event", ev)
            if len(it) > 5 and it[5] is not None:
                d.ready_flag = it[5]
        ids = (C.c_uint64 * max(n, 1))()
        self._check(self._L.kl_submit_batch(self._h, arr, n, ids))
        out = list(ids)[:n]
        for kid, it in zip(out, items):
            self._keep[kid] = it[2]
        return out

    def slice(self, kid: int, blocks_per_sm: int, slice_blocks: int = 0) -> SlicePlan:
        p = SlicePlan()
        self._check(self._L.kl_slice(self._h, kid, blocks_per_sm, slice_blocks, C.byref(p)))
        return p

    def predict(self, cands) -> list[Prediction]:
        n = len(cands)
        arr = (Candidate * max(n, 1))()
        for i, (k1, k2, b1, b2) in enumerate(cands):
            arr[i] = Candidate(KIND_ID[k1] if isinstance(k1, str) else k1,
                               KIND_ID[k2] if isinstance(k2, str) else k2, b1, b2)
        out = (Prediction * max(n, 1))()
        self._check(self._L.kl_predict(self._h, arr, n, out))
        return list(out)[:n]

    def schedule(self) -> CoSchedule | None:
        cs = CoSchedule()
        st = self._L.kl_schedule(self._h, C.byref(cs))
        if st == KL_ENOTFOUND:
            return None
        self._check(st)
        return cs

    def decide(self) -> CoSchedule:
        cs = CoSchedule()
        self._check(self._L.kl_decide(self._h, C.byref(cs)))
        return cs

    def sync(self) -> Counters:
        c = Counters()
        self._check(self._L.kl_sync(self._h, C.byref(c)))
        self._keep.clear()
        return c

    def run_plain(self, kind, grid_blocks: int, args, stream=0, offset: int = 0, n_blocks: int | None = None):
        kid = KIND_ID[kind] if isinstance(kind, str) else int(kind)
        d = KernelDesc(kid, grid_blocks, C.cast(C.pointer(args), _vp), C.sizeof(args), None, 0, None)
        s = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        n = grid_blocks - offset if n_blocks is None else n_blocks
        self._check(self._L.kl_run_plain(self._h, C.byref(d), s, offset, n))

    def run_capped(self, kind, grid_blocks: int, args, cap: int, spin_ns: int = 0) -> float:
        """Whole kernel through the persistent launcher at `cap` blocks/SM; returns device ms
        (spin_ns > 0: that long a device delay precedes the launch inside the timed interval)."""
        kid = KIND_ID[kind] if isinstance(kind, str) else int(kind)
        d = KernelDesc(kid, grid_blocks, C.cast(C.pointer(args), _vp), C.sizeof(args), None, 0, None)
        ms = C.c_double()
        if spin_ns:
            os.environ["KL_TIMING_SPIN_NS"] = str(int(spin_ns))
        try:
            self._check(self._L.kl_run_capped(self._h, C.byref(d), cap, C.byref(ms)))
        finally:
            os.environ.pop("KL_TIMING_SPIN_NS", None)
        return ms.value

    def run_pair(self, kind1, grid1, args1, cap1, kind2, grid2, args2, cap2):
        """Co-run two kernels at the given caps until the first runs out of blocks (the other is
        stopped at its slice boundary); returns the two launch records."""
        k1 = KIND_ID[kind1] if isinstance(kind1, str) else int(kind1)
        k2 = KIND_ID[kind2] if isinstance(kind2, str) else int(kind2)
        d1 = KernelDesc(k1, grid1, C.cast(C.pointer(args1), _vp), C.sizeof(args1), None, 0, None)
        d2 = KernelDesc(k2, grid2, C.cast(C.pointer(args2), _vp), C.sizeof(args2), None, 0, None)
        out = (TraceRec * 2)()
        self._check(self._L.kl_run_pair(self._h, C.byref(d1), cap1, C.byref(d2), cap2, out))
        return out[0], out[1]

    def get_profile(self, kind) -> Profile:
        p = Profile()
        self._check(self._L.kl_get_profile(self._h, KIND_ID[kind] if isinstance(kind, str) else kind, C.byref(p)))
        return p

    def set_profile(self, kind, prof) -> None:
        p = profile_from_dict(prof) if isinstance(prof, dict) else prof
        self._check(self._L.kl_set_profile(self._h, KIND_ID[kind] if isinstance(kind, str) else kind, C.byref(p)))

    def cache_put(self, items):
        """items: [((k1, k2, b1, b2), {ipc1, ipc2, c, solo1, solo2, cp, dT, status})]"""
        n = len(items)
        ca = (Candidate * max(n, 1))()
        pr = (Prediction * max(n, 1))()
        for i, ((k1, k2, b1, b2), d) in enumerate(items):
            ca[i] = Candidate(KIND_ID[k1] if isinstance(k1, str) else k1, KIND_ID[k2] if isinstance(k2, str) else k2, b1, b2)
            for f in ("ipc1", "ipc2", "c", "solo1", "solo2", "cp", "dT", "status"):
                setattr(pr[i], f, d.get(f, 0))
        self._check(self._L.kl_cache_put(self._h, ca, pr, n))

    def reset_model_cache(self):
        self._check(self._L.kl_reset_model_cache(self._h))

    def reset_counters(self):
        self._check(self._L.kl_reset_counters(self._h))

    def trace(self) -> list[TraceRec]:
        n = C.c_size_t()
        self._check(self._L.kl_trace(self._h, None, 0, C.byref(n)))
        arr = (TraceRec * max(n.value, 1))()
        self._check(self._L.kl_trace(self._h, arr, n.value, C.byref(n)))
        return list(arr)[: n.value]

    def stats(self) -> Stats:
        s = Stats()
        self._check(self._L.kl_stats_get(self._h, C.byref(s)))
        return s

    def audit(self, kid: int, n: int):
        """Per-virtual-block execution counts of kernel `kid` (coverage audit)."""
        import numpy as np
        out = np.zeros(n, dtype=np.uint32)
        self._check(self._L.kl_audit(self._h, kid, out.ctypes.data_as(C.POINTER(C.c_uint32)), n))
        return out

    def timeline(self, kid: int, grid: int):
        """(start, end) per block, globaltimer ns (0 = never ran), of kernel `kid` (config audit=2):
        an int64 array of shape (grid, 2)."""
        import numpy as np
        out = np.zeros(2 * grid, dtype=np.uint64)
        self._check(self._L.kl_timeline(self._h, kid, out.ctypes.data, 2 * grid))
        return out.astype(np.int64).reshape(grid, 2)


def profile_dict(p: Profile) -> dict:
    return {name: getattr(p, name) for name, _ in Profile._fields_}

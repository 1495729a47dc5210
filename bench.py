#!/usr/bin/env python
"""Kernel-queue throughput of the B200-native Kernelet hot path (BASELINE.json metric).

One step = one pass of the whole hot path over one batch of synthetic input: submit the queue
(Alg.1 l.2-3), per-kind profiles, pruning, the batched Markov model on the device (the model
cache is cleared every step so the model runs every step), greedy selection, sliced co-scheduled
execution on two lanes with offset-remapped persistent blocks, completion counters, and for N > 1
the NCCL all-gather of the per-GPU counters.

Default workload (N=1): BASELINE configs[1] -- the paper's eight-kernel ALL mix (tb:workloads,
P:1196) at paper sizes (tb:description), 4 instances of each kernel = 32 kernels per
GPU, round-robin arrival order, all pending at t=0.  For N GPUs each rank runs its
own shard of a 32*N-kernel queue (mix-preserving round robin): weak scaling, no cross-GPU data.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
        torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")   # before any CUDA context (see package)

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import kl_inputs as G  # noqa: E402

ALL = G.MIXES["ALL"]
METRIC = "kernel-queue throughput (kernels/s) & speedup vs sequential, 1/2/4/8 B200"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="GPUs (ranks) of this node; without WORLD_SIZE in the environment and N > 1, bench.py "
                         "re-launches itself under torch.distributed.run with N ranks (default: WORLD_SIZE, else 1)")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kernelet", choices=["kernelet", "reference"])
    ap.add_argument("--instances", type=int, default=4, help="instances of each ALL-mix kernel per GPU (c2)")
    ap.add_argument("--workload", default="c5", choices=["c2", "c4", "c5"],
                    help="c5: the 10,000-kernel multi-user queue shared by all GPUs (configs[4], the metric's "
                         "1/2/4/8-GPU workload, strong scaling; default); c4: 1000 random kernels per GPU from "
                         "--mix (configs[3]); c2: the ALL mix x --instances per GPU (configs[1])")
    ap.add_argument("--mix", default="ALL", choices=["ALL", "CI", "MI", "MIX"],
                    help="c4 only: the tb:workloads mix the 1000 kernels are drawn from (P:1193-1196)")
    ap.add_argument("--pool", type=int, default=4,
                    help="input/output sets per kind: instance j of a kind reads input set j %% pool and writes "
                         "output set j %% pool (distinct device buffers)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: functional check of the multi-rank path, "
                         "counters gathered through host memory)")
    ap.add_argument("--size", default="paper", choices=["paper", "small"])
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--profile", default=os.path.join(ROOT, "profiles", "kl_profile_b200.json"))
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--split-rule", type=int, default=1,
                    help="slice ratio per pair: 1 argmax CP over all co-schedules (FindCoSchedule l.3-4, "
                         "default), 0 argmin dT (Eq.8 balanced ratio)")
    ap.add_argument("--cp-min", type=float, default=None)
    ap.add_argument("--alpha", type=float, nargs=2, default=None, metavar=("AP", "AM"),
                    help="pruning thresholds alpha_p alpha_m (default: the profile JSON's, else the paper's 0.4 0.1)")
    ap.add_argument("--age-limit-us", type=int, default=None,
                    help="starvation guard (kl_config.age_limit_us; default 0 = the paper's greedy)")
    ap.add_argument("--levels", default=None, choices=["all", "four"],
                    help="occupancy levels per kernel (kl_config.level_mode): every b with whole warps per virtual "
                         "SM, or the four levels {1/4, 1/2, 3/4, 1} x b_max of config C2 (default: four for c2, "
                         "all for c4/c5, whose configs fix no levels: C5 3442-3452 vs 3401-3411 kernels/s)")
    ap.add_argument("--speculative", action="store_true", help="enable the speculative start (kl_config.speculative)")
    ap.add_argument("--critical", type=int, default=0, choices=[0, 1],
                    help="1: makespan extension of FindCoSchedule (kl_config.critical, reading R29): while one kind's "
                         "predicted remaining solo time exceeds all others' together, only co-schedules with it")
    ap.add_argument("--bmax", default="hw", choices=["sat", "hw"],
                    help="b_max with every whole-warp level: the hardware limit (default) or the calibrated "
                         "saturation occupancy with distinct-kind pairs (R31/R31b, measured option)")
    ap.add_argument("--prof", action="append", default=[], metavar="KIND.FIELD=VALUE",
                    help="A/B knob: override one field of a kind's profile (e.g. MRIQ.bmax=3)")
    ap.add_argument("--set", action="append", default=[], metavar="FIELD=VALUE",
                    help="A/B knob: set a kl_config integer/float field (e.g. model_states=3, granularity=1)")
    ap.add_argument("--trace-out", default=None, help="write the last timed step's launch trace (JSON lines)")
    ap.add_argument("--opt", default=None, help="OPT comparator: decide from a measured pair table "
                                               "(tools/opt_table.py) instead of the Markov model")
    return ap.parse_args(argv)


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_cmd(args, argv: list[str]) -> list[str] | None:
    """The torch.distributed.run command that re-launches this script with args.gpus ranks, or None
    when no spawn is needed (already under a launcher, N = 1, or the reference arm, which runs on
    rank 0 only)."""
    if "WORLD_SIZE" in os.environ or args.impl == "reference" or (args.gpus or 1) <= 1:
        return None
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + list(argv)


# ---------------------------------------------------------------------------------------------
# Algorithmic work per kernel: bytes that must cross HBM, or the
# arithmetic the method must do, per instance at the given size.  Used for the roofline.
# ---------------------------------------------------------------------------------------------
def algorithmic_work(kind: str, p: dict) -> dict:
    if kind == "PC":      # one 64-B HBM3e access per random dependent load (nodes are visited
        # once: no reuse for L2) + 8 B of output per thread; ncu: 64 B DRAM read per hop
        # (DESIGN reading R27: the HBM3e access atom is 64 B; SURVEY §8(d)'s 32-B-sector figure
        # is reported beside it as bytes_32B)
        return {"bound": "hbm", "bytes": p["n_threads"] * (p["hops"] * 64 + 8),
                "bytes_32B": p["n_threads"] * (p["hops"] * 32 + 8)}
    if kind == "SAD":     # 4 pixel |diff|-accumulates per vabsdiff4; ALU-bound
        n_mb = (p["width"] // 16) * (p["height"] // 16)
        return {"bound": "alu", "ops": n_mb * 1089 * 256 / 4, "bytes": 2 * p["width"] * p["height"] + n_mb * 1089 * 2}
    if kind == "SPMV":
        nnz = p["n_rows"] * (p["nnz_min"] + p["nnz_max"]) / 2
        return {"bound": "hbm", "bytes": nnz * 8 + (p["n_rows"] + 1) * 4 + p["n_cols"] * 4 + p["n_rows"] * 4}
    if kind == "ST":
        return {"bound": "hbm", "bytes": 2 * 4 * p["nx"] * p["ny"] * p["nz"]}
    if kind == "MM":
        return {"bound": "tensor", "flops": 2.0 * p["M"] * p["N"] * p["K"],
                "bytes": 2 * (p["M"] * p["K"] + p["N"] * p["K"]) + 4 * p["M"] * p["N"]}
    if kind == "MRIQ":    # sin + cos per (voxel, k): MUFU-bound
        return {"bound": "alu", "ops": 2.0 * p["num_x"] * p["num_k"], "bytes": 5 * 4 * p["num_x"]}
    if kind == "BS":
        return {"bound": "hbm", "bytes": 5 * 4 * p["n"]}
    if kind == "TEA":     # 32 cycles x ~10 integer ops per 64-bit block
        return {"bound": "alu", "ops": p["n"] * 32 * 2 * 5.0, "bytes": 16 * p["n"]}
    return {"bound": "hbm", "bytes": 0}


_UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def _metric_bytes(m: dict) -> float:
    """One ncu raw-page metric {"value": "1,234.5", "unit": "Mbyte"} in bytes (each metric carries
    its own unit: ncu scales read and write bytes independently)."""
    return float(str(m["value"]).replace(",", "")) * _UNIT[m.get("unit", "byte")]


def ncu_traffic(kind: str, profiles_dir: str | None = None):
    """DRAM bytes (read + write) of one launch of `kind` from the committed `ncu --set full`
    summary (profiles/*ncu_summary.json, latest round), or None."""
    import glob
    pdir = profiles_dir or os.path.join(ROOT, "profiles")
    for path in sorted(glob.glob(os.path.join(pdir, "r*_ncu_summary.json")), reverse=True):
        try:
            d = json.load(open(path))
        except Exception:
            continue
        rows_all = [r for rows in d.values() if isinstance(rows, list) for r in rows]
        # the persistent slice-launcher variant first: that is what the bench's step launches
        rows_all.sort(key=lambda r: 0 if "k_persistent" in r.get("kernel", "") else 1)
        for rows in (rows_all,):
            for r in rows:
                if f"Body{kind}>" in r.get("kernel", "") or f"Body{kind}E" in r.get("kernel", "") or \
                        f"::Body{kind}" in r.get("kernel", "") or f"Body{kind}<" in r.get("kernel", ""):
                    try:
                        rd = _metric_bytes(r["dram__bytes_read.sum"])
                        wr = _metric_bytes(r["dram__bytes_write.sum"])
                        return {"bytes_per_instance": rd + wr, "read": rd, "write": wr,
                                "source": os.path.basename(path)}
                    except (KeyError, ValueError):
                        continue
    return None


def pipe_peaks() -> dict:
    """Builder-measured lane ops per SM clock (tools/pipe_peaks.cu -> profiles/r*_pipe_peaks.json,
    latest round); the guide's nominal unit counts where a pipe was not measured."""
    import glob
    out = {"mufu_sincos": (16.0, "nominal"), "vabsdiff4": (64.0, "nominal"), "issue": (128.0, "nominal")}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_pipe_peaks.json")), reverse=True):
        try:
            d = json.load(open(path))
        except Exception:
            continue
        for k in ("mufu_sincos", "vabsdiff4"):
            if k in d:
                out[k] = (float(d[k]["lane_ops_per_clk_per_sm"]), f"builder-measured ({os.path.basename(path)})")
        if "ffma" in d and "imad" in d:       # TEA issues on the alu and fma pipes together
            out["issue"] = (float(d["imad"]["lane_ops_per_clk_per_sm"]) + float(d["lop3"]["lane_ops_per_clk_per_sm"]),
                            f"builder-measured IMAD + LOP3 pipes ({os.path.basename(path)})")
        break
    return out


def alu_peak(kind: str, sm_mhz: float, n_sm: int = 148) -> tuple[float, str]:
    """ALU peaks from lane ops per SM clock x SMs x clock: MRIQ's sin + cos on
    MUFU; SAD's VABSDIFF4 on the alu pipe; TEA's integer mix spread over the alu pipe (IADD3/LOP3/
    SHF) and the fma pipe (IMAD), so its ceiling is the two pipes together."""
    f = sm_mhz * 1e6
    pp = pipe_peaks()
    key = {"MRIQ": "mufu_sincos", "TEA": "issue"}.get(kind, "vabsdiff4")
    per, src = pp[key]
    label = {"MRIQ": "MUFU ops/s", "TEA": "int ops/s (alu+fma pipes)"}.get(kind, "int ALU ops/s")
    return per * n_sm * f, f"{label} ({per:.2f}/clk/SM, {src})"


# ---------------------------------------------------------------------------------------------
class Clocks:
    """Sample nvidia-smi during the timed region (B200_PROFILING.md clocks line): one streaming
    `nvidia-smi -lms 100` process started before and stopped after the timed steps."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "100"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        time.sleep(0.2)
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=5)
        except Exception:
            self._p.kill()
            out, _ = self._p.communicate()
        for line in out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 8:
                self.samples.append(f)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 4 + i and "Active" in s[4 + i]
                          and s[4 + i].strip() == "Active"})
        loaded = [x for x in sm if x > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------------------------
def global_queue(workload: str, instances: int, world: int, mix: str = "ALL") -> list[str]:
    """c2 (configs[1]): ALL mix, `instances` of each kernel per GPU, round-robin arrivals.
    c4 (configs[3]): 1000 kernels per GPU drawn uniformly from `mix` (ALL, or the CI/MI/MIX
    variants of tb:workloads; seed 42).
    c5 (configs[4]): 10,000-kernel multi-user queue (16 Poisson users on CI/MI/MIX/ALL), the
    whole queue shared by all GPUs (strong scaling)."""
    if workload == "c2":
        return [e["kind"] for e in G.queue("ALL", len(ALL) * instances * world, order="round_robin")]
    if workload == "c4":
        return [e["kind"] for e in G.queue(mix, 1000 * world, seed=42, order="uniform")]
    if workload == "c5":
        return [e["kind"] for e in G.multi_user_queue(10000, 16, seed=7)]
    raise ValueError(workload)


def build_queue(rank: int, world: int, instances: int, workload: str = "c5", mix: str = "ALL") -> list[str]:
    """This GPU's shard of the global queue, mix-preserving round robin."""
    from paper_1303_5164_b200.dist import shard
    return shard(global_queue(workload, instances, world, mix), rank, world)


MODEL_FIELDS = ("rm", "r", "ipb", "pur", "mur", "m_min", "ipc_max", "pipe", "uc", "ru")


def load_profiles(path: str, levels: str = "four", bmax: str = "hw"):
    """Calibrated model inputs (tools/calibrate.py).  Resource fields (warps, registers, shared
    memory, TMEM, b_max) are left to the runtime, which reads them from the compiled kernels --
    except that with every whole-warp level (C4 / C5, `levels="all"`) and `bmax="sat"` b_max is
    the kind's saturation occupancy `bmax_sat` (reading R31: the smallest cap whose solo time is
    within 1 % of the best in the calibration's occupancy sweep; a measured option, not the
    default).  C2 fixes its levels as quarters of the hardware b_max and keeps it."""
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        profs = {k: {f: v[f] for f in MODEL_FIELDS if f in v} for k, v in d.get("profiles", {}).items()}
        if levels == "all" and bmax == "sat":
            for k, v in d.get("profiles", {}).items():
                if v.get("bmax_sat"):
                    profs[k]["bmax"] = int(v["bmax_sat"])
        return profs, d.get("config", {})
    return None, {}


def max_over_ranks(x: float, dev, world: int, backend: str = "nccl") -> float:
    """The slowest rank's value (whole-job time is set by the last GPU to finish)."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_kernelet(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1303_5164_b200 as K
    from paper_1303_5164_b200.workload import Instance, inputs_to_device

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    K.lib()
    kinds = build_queue(rank, world, args.instances, args.workload, args.mix)
    profiles, kcfg = load_profiles(args.profile, args.levels, args.bmax)
    for kv in args.prof:
        kf, _, v = kv.partition("=")
        kind, _, field = kf.partition(".")
        profiles.setdefault(kind, {})[field] = float(v) if "." in v else int(v)
    t_gen = time.time()
    data = {k: G.gen(k, args.size) for k in sorted(set(kinds))}
    # leases: POOL input sets and POOL output sets per kind (distinct device buffers; input set j
    # is a device copy of the generated set, so every set has the oracle's values); instance j of
    # a kind reads input set j % POOL and writes output set j % POOL.  The trace check below
    # proves no two launches that were resident at the same time wrote the same output set.
    from paper_1303_5164_b200.workload import alloc_outputs
    POOL = max(1, args.pool)
    in_pools, pools, seen, lease = {}, {}, {}, []
    insts = []
    for k in kinds:
        j = seen.get(k, 0)
        seen[k] = j + 1
        if j < POOL:
            if j == 0:
                in_pools[k] = [inputs_to_device(data[k], dev)]
            else:
                in_pools[k].append({n: t.clone() for n, t in in_pools[k][0].items()})
            pools.setdefault(k, []).append(alloc_outputs(k, data[k]["params"], dev))
        insts.append(Instance(data[k], dev, inputs=in_pools[k][j % POOL], outputs=pools[k][j % POOL]))
        insts[-1].lease = j % POOL
        lease.append((k, j % POOL))
    torch.cuda.synchronize(dev)
    t_gen = time.time() - t_gen
    counters = torch.zeros(8, dtype=torch.int64, device=dev)
    lane_a = torch.cuda.Stream(device=dev)
    lane_b = torch.cuda.Stream(device=dev)
    cfg = dict(kcfg)
    cfg["split_rule"] = args.split_rule
    cfg["level_mode"] = 1 if args.levels == "four" else 0
    if args.alpha:
        cfg["alpha_p"], cfg["alpha_m"] = args.alpha
    if args.speculative:
        cfg["speculative"] = 1
    if args.critical:
        cfg["critical"] = 1
    if args.levels == "all" and args.bmax == "sat":
        cfg["distinct_kinds"] = 1      # R31b: a same-kind pair is the kind above its saturation occupancy
    for kv in args.set:
        k, _, v = kv.partition("=")
        cfg[k] = float(v) if "." in v else int(v)
    if args.age_limit_us is not None:
        cfg["age_limit_us"] = args.age_limit_us
    if args.cp_min is not None:
        cfg["cp_min"] = args.cp_min
    if args.opt:
        cfg["model_frozen"] = 1
    ctx = K.Context(device=local_rank, profiles=profiles, streams=(lane_a, lane_b), counters=counters, **cfg)
    if args.opt:   # the paper's OPT: the same greedy Alg.1 over pre-executed (measured) CP
        tab = json.load(open(args.opt))["table"]
        ctx.cache_put([((t["k1"], t["k2"], t["b1"], t["b2"]), t) for t in tab])
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > L2 (126.5 MiB)
    nccl = world > 1 and args.backend == "nccl"
    gathered = torch.zeros(world * 8, dtype=torch.int64, device=dev if nccl else "cpu")

    counters[5] = rank      # kl_counters.rank / .world: the per-step reset clears fields 0-4 only
    counters[6] = world

    def one_step():
        if not args.opt:
            ctx.reset_model_cache()
        ctx.reset_counters()
        ids = ctx.submit_many([(i.kind, i.grid, i.args, n + 1, None) for n, i in enumerate(insts)])
        c = ctx.sync()
        if nccl:        # the one collective: per-GPU counters, read by NCCL from device memory
            with torch.cuda.stream(lane_a):
                dist.all_gather_into_tensor(gathered, counters)
        elif world > 1:
            dist.all_gather_into_tensor(gathered, counters.cpu())
        return ids, c

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # warm-up (also the parity sample of this run)
    for _ in range(args.warmup):
        flush.zero_()
        barrier()
        one_step()
    torch.cuda.synchronize(dev)
    parity = sample_parity(insts, data) if rank == 0 else {}
    n_trace0 = len(ctx.trace())

    step_ms, dev_ms, cnts = [], [], []
    dec0 = ctx.stats().decisions
    dl0 = ctx.stats().device_launches
    with Clocks(local_rank) as clk:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(lane_a)
            ids, c = one_step()
            e1.record(lane_a)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            dev_ms.append((c.t_end_ns - c.t_start_ns) / 1e6)
            cnts.append(c)
        barrier()
    trace = ctx.trace()[n_trace0:]
    st = ctx.stats()
    # per kind inside the timed region (device launch records, %globaltimer): blocks executed and
    # the union of the intervals in which a launch of the kind was resident
    timed = {}
    for k in sorted(set(i.kind for i in insts)):
        iv = sorted((t.t0_ns, t.t1_ns) for t in trace if K.KINDS[t.kind] == k and t.admitted)
        busy, cur0, cur1 = 0, None, None
        for a, z in iv:
            if cur1 is None or a > cur1:
                if cur1 is not None:
                    busy += cur1 - cur0
                cur0, cur1 = a, z
            else:
                cur1 = max(cur1, z)
        if cur1 is not None:
            busy += cur1 - cur0
        timed[k] = {"blocks": sum(t.executed for t in trace if K.KINDS[t.kind] == k),
                    "busy_ms": busy / 1e6, "launches": len(iv)}
    launches = st.device_launches - dl0         # slice grids, top-ups, model batches, ctl inits
    if args.trace_out and rank == 0:
        last = trace[-max(1, len(trace) // args.steps):]
        z = min(t.t0_ns for t in last if t.admitted)
        with open(args.trace_out, "w") as f:
            for t in sorted(last, key=lambda t: t.t0_ns):
                f.write(json.dumps({"kind": K.KINDS[t.kind], "cap": t.cap, "cap_max": t.cap_max, "grids": t.grids,
                                    "start": t.start, "end": t.end, "exh": t.exhausted, "adm": t.admitted, "mx": t.max_per_sm,
                                    "t0_us": round((t.t0_ns - z) / 1e3, 1), "t1_us": round((t.t1_ns - z) / 1e3, 1),
                                    "partner": K.KINDS[t.partner_kind] if t.partner_kind >= 0 else None,
                                    "cp": round(t.cp, 3), "dec": t.phase}) + "\n")
    lease_conflicts = check_leases(trace, ids, lease)
    total_ms = max_over_ranks(sum(step_ms), dev, world, args.backend)
    c_last = cnts[-1]
    assert c_last.kernels_done == len(insts), (c_last.kernels_done, len(insts))
    n_done = len(insts)
    if world > 1:       # whole-job completion from the all-gathered counters of the last step
        g = gathered.view(world, 8).cpu()
        n_done = int(g[:, 0].sum())
        assert [int(x) for x in g[:, 6]] == [world] * world and sorted(int(x) for x in g[:, 5]) == list(range(world))
        assert n_done == args.n_global, (n_done, args.n_global)
    res = {
        "value": n_done * args.steps / (total_ms / 1e3),
        "kernels_per_rank": len(insts),
        "ms_per_step": total_ms / args.steps,
        "device_ms_per_step": statistics.median(dev_ms),
        "phases_per_step": (ctx.stats().decisions - dec0) / args.steps,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "parity": parity,
        "setup_s": round(t_gen, 1),
        "lease_conflicts": lease_conflicts,
        "timed_kernels": timed,
        "retunes_per_step": st.retunes / max(1, args.warmup + args.steps),
        "stops_per_step": st.stops / max(1, args.warmup + args.steps),
        "memops_per_step": st.memops / max(1, args.warmup + args.steps),
        "host_decide_ms_per_step": st.decide_ns / 1e6 / max(1, args.warmup + args.steps),
        "model_ms_per_step": st.model_ns / 1e6 / max(1, args.warmup + args.steps),
    }
    phase_kinds = [(K.KINDS[tr.kind], tr.cap, K.KINDS[tr.partner_kind] if tr.partner_kind >= 0 else None)
                   for tr in trace[: max(1, len(trace) // args.steps)]]
    res["schedule_first_step"] = phase_kinds

    if not args.no_baselines:
        res["baselines"] = baselines(ctx, insts, dev, flush, barrier, args, world)
        res["per_kernel"] = per_kernel(ctx, insts, data, dev, flush, barrier)
        res["e2e"] = e2e(ctx, insts, data, dev, barrier, args, world, rank, lane_a, lane_b, res["per_kernel"])
    ctx.close()
    return res


def check_leases(trace, ids, lease) -> int:
    """Launches of different instances that share an output set must never be resident at the
    same time (per-launch [t0, t1] from the device records)."""
    owner = {kid: lease[n] for n, kid in enumerate(ids)}
    spans = {}
    for t in trace:
        if t.id in owner and t.admitted:
            spans.setdefault(owner[t.id], []).append((t.t0_ns, t.t1_ns, t.id))
    bad = 0
    for v in spans.values():
        v.sort()
        for (a0, a1, ia), (b0, b1, ib) in zip(v, v[1:]):
            if ia != ib and b0 < a1:
                bad += 1
    return bad


def sample_parity(insts, data, per_kind: int = 64) -> dict:
    """Sampled outputs of every kind vs the oracle at full size (tests/kl_check tolerances)."""
    import oracle as O
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from kl_check import compare
    out, seen = {}, set()
    rng = np.random.default_rng(5)
    for inst in insts:
        k = inst.kind
        if k in seen:
            continue
        seen.add(k)
        res = inst.result()
        first = next(iter(res.values()))
        n = first.size if k != "TEA" else first.size // 2
        idx = np.sort(rng.choice(n, size=min(per_kind, n), replace=False))
        ref = O.run_kernel(data[k], idx)
        try:
            errs = compare(k, res, ref, idx=idx)
            out[k] = {"ok": True, "max_err": max(errs.values()) if errs else 0.0, "n": int(idx.size)}
        except AssertionError as e:
            out[k] = {"ok": False, "err": str(e)[:200]}
    return out


def _time_streams(fn, dev, flush, barrier, reps=3, pre=None):
    """Device time of fn's launches between two events on the current stream, L2 flushed before
    each rep.  pre(s), if given, is enqueued before the first event (a device-side delay that keeps
    the host's launch latency out of a single short kernel's interval)."""
    import torch
    ts = []
    for _ in range(reps):
        flush.zero_()
        barrier()
        s = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if pre is not None:
            pre(s)
        e0.record(s)
        fn(s, e0)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def baselines(ctx, insts, dev, flush, barrier, args, world=1) -> dict:
    """Sequential (one stream, full grids at max occupancy, back to back) and plain multi-stream
    (round robin over S streams, full grids, no slicing) executions of the same kernels, on every
    rank's shard; whole-job time = the slowest rank."""
    import torch
    out = {}
    n = args.n_global

    def seq(s, e0):
        for i in insts:
            ctx.run_plain(i.kind, i.grid, i.args, s)

    ms = max_over_ranks(_time_streams(seq, dev, flush, barrier), dev, world, args.backend)
    out["sequential"] = {"ms_per_step": ms, "kernels_per_s": n / (ms / 1e3)}
    for S in (2, 4, 8):
        streams = [torch.cuda.Stream(device=dev) for _ in range(S)]

        def ms_fn(s, e0, streams=streams):
            for st in streams:
                st.wait_event(e0)
            for j, i in enumerate(insts):
                ctx.run_plain(i.kind, i.grid, i.args, streams[j % len(streams)])
            for st in streams:
                ev = torch.cuda.Event()
                ev.record(st)
                s.wait_event(ev)

        ms = max_over_ranks(_time_streams(ms_fn, dev, flush, barrier), dev, world, args.backend)
        out[f"multistream{S}"] = {"ms_per_step": ms, "kernels_per_s": n / (ms / 1e3)}
    return out


def per_kernel(ctx, insts, data, dev, flush, barrier) -> dict:
    """Solo plain launch of one instance of each kind: duration, algorithmic rate, roofline."""
    import torch
    out, seen = {}, set()
    for i in insts:
        if i.kind in seen:
            continue
        seen.add(i.kind)
        # the GPU is idle after the barrier: without a device-side delay before the first event the
        # interval would include the host's launch path (~10-17 us, 25 % of MM's 60 us)
        ms = _time_streams(lambda s, e0, i=i: ctx.run_plain(i.kind, i.grid, i.args, s), dev, flush, barrier, reps=5,
                           pre=lambda s: ctx.delay(s, 200_000))
        w = algorithmic_work(i.kind, data[i.kind]["params"])
        out[i.kind] = {"ms": ms, "grid": i.grid, **w}
    return out


def johnson_order(jobs, a, b):
    """Johnson's rule for a two-machine flow shop (machine 1 = the H2D copy stream, machine 2 = the
    GPU's kernels): jobs with a < b first by increasing a, then the rest by decreasing b; minimises
    the makespan of the two-stage pipeline."""
    first = sorted((j for j in jobs if a[j] < b[j]), key=lambda j: a[j])
    rest = sorted((j for j in jobs if a[j] >= b[j]), key=lambda j: -b[j])
    return first + rest


def e2e(ctx, insts, data, dev, barrier, args, world, rank, lane, lane_b, pk=None) -> dict:
    """Same metric through the public API with HOST buffers.  Every step copies every input set
    of the step (the --pool sets per kind; instance j of a kind reads set j % pool) from pinned
    host memory and reads every output set back (the last instance written to each set), inside
    the timed region.  Each input set's copy is the arrival of the kernels that read it: they are
    submitted with the copy's event as `ready_event`, so the scheduler overlaps the PCIe transfer
    of later sets with the execution of earlier ones (arrivals trigger re-planning)."""
    import torch
    sets = []               # (kind, lease) in first-use order
    for i in insts:
        if (i.kind, i.lease) not in sets:
            sets.append((i.kind, i.lease))
    rep = {s: next(i for i in insts if (i.kind, i.lease) == s) for s in sets}
    # copy order: a two-stage flow shop (one copy stream, then the kernels), ordered by Johnson's
    # rule -- sets whose copy is shorter than their kernel time first, by increasing copy time;
    # then the rest by decreasing kernel time -- so the last copy has the least kernel time behind
    # it (copy time from the bytes at the measured ~55 GB/s pinned H2D rate)
    if pk:
        nk = {s: sum(1 for i in insts if (i.kind, i.lease) == s) for s in sets}
        a = {s: rep[s].input_bytes() / 55e9 * 1e3 for s in sets}
        b = {s: pk[s[0]]["ms"] * nk[s] for s in sets}
        sets = johnson_order(sets, a, b)
    host_in = {s: {n: t.cpu().pin_memory() for n, t in rep[s].inputs.items()} for s in sets}
    host_out = {s: {n: torch.empty_like(t, device="cpu").pin_memory() for n, t in rep[s].outputs.items()}
                for s in sets}
    h2d = sum(t.numel() * t.element_size() for d in host_in.values() for t in d.values())
    d2h = sum(t.numel() * t.element_size() for d in host_out.values() for t in d.values()) + 64
    copy_stream = torch.cuda.Stream(device=dev)
    ts = []
    for _ in range(max(2, min(args.steps, 3))):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(lane)
        copy_stream.wait_event(e0)
        ready = {}
        with torch.cuda.stream(copy_stream):
            for s in sets:
                for n, t in rep[s].inputs.items():
                    t.copy_(host_in[s][n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy_stream)
                ready[s] = ev
        ctx.reset_model_cache()
        ctx.reset_counters()
        ctx.submit_many([(i.kind, i.grid, i.args, n + 1, ready[(i.kind, i.lease)]) for n, i in enumerate(insts)])
        c = ctx.sync()
        with torch.cuda.stream(lane):   # D2H of the step's results: every output set + counters
            for s in sets:
                for n, t in rep[s].outputs.items():
                    host_out[s][n].copy_(t, non_blocking=True)
            res = ctx.counters.to("cpu", non_blocking=True)
        e1.record(lane)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
        assert int(res[0]) == len(insts)
    ms = max_over_ranks(statistics.median(ts), dev, world, args.backend)
    return {"value": args.n_global / (ms / 1e3), "unit": "kernels/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": ms, "h2d_GBps": h2d / (ms / 1e3) / 1e9,
            "copy_order": [f"{k}#{j}" for k, j in sets],
            "what": f"every step: H2D of all {len(sets)} input sets ({args.pool} per kind, pinned host -> device), "
                    f"the queue, D2H of all {len(sets)} output sets + the counters"}


# ---------------------------------------------------------------------------------------------
class OracleLeg:
    """The oracle as it stands, on the host cores: every kind's outputs on a fixed strided sample
    (fraction f of the elements) plus the oracle's Alg.1 decision sequence for the queue, run in
    the GPU run's configuration (the calibrated profile's L0/B/a0/b0 latency, alpha_p/alpha_m, the
    occupancy-level mode and the split rule); throughput = kernels-equivalent of work done / wall
    time."""

    def __init__(self, kinds: list[str], size: str, profile_path: str | None = None, split_rule: int = 1,
                 levels: str = "four", alpha=None, max_decisions: int = 200, cp_min=None, bmax: str = "hw"):
        import oracle as O
        O.build()
        self.O = O
        self.kinds = kinds
        self.cores = os.cpu_count() or 1
        self.data = {k: G.gen(k, size) for k in sorted(set(kinds))}
        self.sizes = {}
        for k, d in self.data.items():
            p = d["params"]
            self.sizes[k] = {"PC": lambda: p["n_threads"], "SPMV": lambda: p["n_rows"], "MRIQ": lambda: p["num_x"],
                             "BS": lambda: p["n"], "TEA": lambda: p["n"],
                             "SAD": lambda: (p["width"] // 16) * (p["height"] // 16) * 1089,
                             "ST": lambda: p["nx"] * p["ny"] * p["nz"], "MM": lambda: p["M"] * p["N"]}[k]()
        self.profs, pcfg = _oracle_profiles(profile_path, levels, bmax)
        self.cfg = O.smcfg(L0=pcfg.get("L0", 800.0), B=pcfg.get("B", 1.0), a0=pcfg.get("a0", 0.0),
                           b0=pcfg.get("b0", 0.0), W=16)
        ap, am = alpha if alpha else (pcfg.get("alpha_p", 0.4), pcfg.get("alpha_m", 0.1))
        self.sched_kw = dict(ap=ap, am=am, mode="4" if levels == "four" else "all", split_rule=split_rule,
                             cp_min=pcfg.get("cp_min", 0.0) if cp_min is None else cp_min,
                             distinct_kinds=levels == "all" and bmax == "sat")
        self.max_decisions = max_decisions
        self.config = {"L0": self.cfg.L0, "B": self.cfg.B, "a0": self.cfg.a0, "b0": self.cfg.b0, "W_v": 16,
                       **self.sched_kw}

    def run(self, target_s: float) -> dict:
        frac = 1e-4          # grow the sample until it takes about target_s (bounded CPU work)
        while True:
            t_kind = _oracle_sample(self.O, self.data, self.sizes, frac, self.cores)
            t_k = sum(t_kind.values())
            if t_k >= 0.5 * target_s or frac >= 1.0:
                break
            frac = min(1.0, frac * min(20.0, target_s / max(t_k, 1e-3)))
        t0 = time.time()
        n_dec = 0
        if self.profs:
            # the decision sequence for the first max_decisions queue entries (each decision
            # searches every pending kind pair, so its cost does not depend on the queue length
            # once all kinds are pending)
            q = [{"kind": k, "blocks": 1000} for k in self.kinds[: self.max_decisions]]
            _, tr = self.O.alg1_makespan(q, self.profs, self.cfg, **self.sched_kw)
            n_dec = len(tr)
        t_s = time.time() - t0
        # whole-queue oracle time: each kind's sampled time scaled to one full instance, times the
        # kind's count in the queue, plus the decisions scaled to one per kernel
        count = {k: self.kinds.count(k) for k in t_kind}
        t_queue = sum(count[k] * t_kind[k] / frac for k in t_kind) + t_s * len(self.kinds) / max(1, n_dec)
        return {"value": len(self.kinds) / t_queue, "unit": "kernels/s", "cores": self.cores, "kind": "oracle",
                "sample": f"{frac:.2e} of the output elements of one instance of each of the {len(t_kind)} kinds "
                          f"(strided, {self.cores} threads, {t_k:.1f} s), scaled to the {len(self.kinds)}-kernel "
                          f"queue's kind counts, + the oracle's Alg.1/FindCoSchedule decisions for the first "
                          f"{min(len(self.kinds), self.max_decisions) if self.profs else 0} kernels ({n_dec} decisions, "
                          f"{t_s:.1f} s; charged per kernel) in the GPU run's model configuration {self.config}"}


def cpu_oracle_leg(kinds: list[str], size: str, target_s: float = 15.0, **kw) -> dict:
    return OracleLeg(kinds, size, **kw).run(target_s)


def _oracle_sample(O, data, sizes, frac, cores) -> dict:
    """Run the oracle on a strided `frac` of every kind's output elements, the kind's elements
    split over `cores` threads; returns wall seconds per kind."""
    from concurrent.futures import ThreadPoolExecutor
    out = {}
    with ThreadPoolExecutor(cores) as ex:
        for k, d in data.items():
            n = sizes[k]
            m = max(1, int(n * frac))
            idx = np.linspace(0, n - 1, m).astype(np.int64)
            t0 = time.time()
            list(ex.map(lambda c, d=d: O.run_kernel(d, c), [c for c in np.array_split(idx, cores) if c.size]))
            out[k] = time.time() - t0
    return out


def profile_label(path: str) -> str:
    """The calibration file the model decides from: its name and calibration time."""
    try:
        with open(path) as f:
            when = json.load(f).get("when", "?")
    except (OSError, ValueError):
        return f"{os.path.basename(path)} (missing: built-in defaults)"
    return f"{os.path.relpath(path, ROOT)} (calibrated {when})"


def _oracle_profiles(path: str | None = None, levels: str = "four", bmax: str = "hw"):
    """The oracle's profile table: the calibrated profiles with the b_max the GPU run uses
    (load_profiles: bmax_sat with every whole-warp level when bmax="sat")."""
    path = path or os.path.join(ROOT, "profiles", "kl_profile_b200.json")
    if not os.path.exists(path):
        return None, {}
    d = json.load(open(path))
    out = {k: dict(v) for k, v in d["profiles"].items() if k in ALL}
    if levels == "all" and bmax == "sat":
        for v in out.values():
            if v.get("bmax_sat"):
                v["bmax"] = int(v["bmax_sat"])
    return out, d.get("config", {})


# ---------------------------------------------------------------------------------------------
def workload_name(args) -> str:
    return {"c2": f"C2: ALL mix x{args.instances} per GPU ({len(ALL) * args.instances} kernels per GPU, {args.size} "
                  "sizes, all pending at t=0)",
            "c4": f"C4: 1000 kernels per GPU uniform over {args.mix} (seed 42), {args.size} sizes",
            "c5": f"C5: 10,000-kernel multi-user queue (16 Poisson users on CI/MI/MIX/ALL, seed 7) shared by all "
                  f"GPUs, {args.size} sizes"}[args.workload]


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.levels is None:
        args.levels = "four" if args.workload == "c2" else "all"
    cmd = spawn_cmd(args, argv)
    if cmd:                 # --gpus N without a launcher: one process per GPU via torch.distributed.run
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.gpus is None:
        args.gpus = world
    if args.impl != "reference" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    args.n_global = len(global_queue(args.workload, args.instances, world, args.mix))
    config = {"workload": workload_name(args), "global_kernels": args.n_global,
              "sizes": "tb:description (million = 2^20), MRIQ numK = 2048", "parallelism": f"queue shard x{world}",
              "l2": "256 MiB write between steps; inputs >> L2", "model_cache": "cleared every step",
              "leases": f"{args.pool} input sets + {args.pool} output sets per kind (distinct device buffers)",
              "split_rule": "argmax CP over (pair, ratio)" if args.split_rule == 1 else "argmin dT (Eq.8)",
              "cp_min": args.cp_min if args.cp_min is not None else load_profiles(args.profile)[1].get("cp_min", 0.0),
              "decisions_from": "measured pair table (OPT)" if args.opt else "Markov model",
              "profile": profile_label(args.profile),
              "pair_choice": "critical-kind restriction (R29)" if args.critical else "max CP (Alg.1 greedy)",
              **({"config_overrides": args.set} if args.set else {}),
              **({"profile_overrides": args.prof} if args.prof else {}),
              "occupancy_levels": "{1/4, 1/2, 3/4, 1} x b_max per kernel (config C2)" if args.levels == "four"
              else ("every b with whole warps per virtual SM up to the kind's saturation occupancy (R31)"
                    if args.bmax == "sat" else "every b with whole warps per virtual SM up to the hardware b_max")}
    scaling = "strong" if args.workload == "c5" else "weak"
    leg_kw = dict(profile_path=args.profile, split_rule=args.split_rule, levels=args.levels, alpha=args.alpha,
                  cp_min=args.cp_min, bmax=args.bmax)

    if args.impl == "reference":
        if rank != 0:
            return
        kinds = build_queue(0, 1, args.instances, args.workload, args.mix)
        leg = OracleLeg(kinds, args.size, **leg_kw)
        vals = []
        for s in range(args.warmup + args.steps):
            r = leg.run(target_s=max(2.0, 60.0 / (args.warmup + args.steps)))
            if s >= args.warmup:
                vals.append(r["value"])
        v = statistics.median(vals)
        line = {"metric": METRIC, "value": v, "unit": "kernels/s", "impl": "reference", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f32/f64/u32 (per kernel)", "data": "synthetic", "config": config,
                "cpu_baseline": {**r, "value": v}, "e2e": {"value": v, "unit": "kernels/s", "h2d_bytes_per_step": 0,
                                                          "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    if os.environ.get("KL_BENCH_ONE_DEVICE"):   # functional multi-rank check on a one-GPU box
        local_rank = 0
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    res = run_kernelet(args, rank, world, local_rank)
    if rank == 0:
        bl = res.get("baselines", {})
        seq = bl.get("sequential", {}).get("kernels_per_s")
        ms4 = max((v["kernels_per_s"] for k, v in bl.items() if k.startswith("multistream")), default=None)
        pk = res.get("per_kernel", {})
        # ALU peaks scale with the SM clock: the solo kernels (timed alone, outside the timed
        # region) against the maximum clock, the in-step roofline against the median clock the
        # nvidia-smi samples saw during the timed steps (sw_power_cap lowers it under the queue)
        sm_mhz = (res["clocks"].get("sm_mhz") or 1965.0)
        sm_max = (res["clocks"].get("sm_max_mhz") or 1965.0)
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
        roof_all = {}
        for k, v in pk.items():
            if v["bound"] == "hbm":
                a = v["bytes"] / (v["ms"] / 1e3) / 1e9
                roof_all[k] = {"bound": "hbm", "achieved": a, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                               "frac": a / peaks["hbm_gbs"], "ms": v["ms"]}
            elif v["bound"] == "tensor":
                a = v["flops"] / (v["ms"] / 1e3) / 1e12
                roof_all[k] = {"bound": "tensor", "achieved": a, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                               "frac": a / peaks["bf16_tflops"], "ms": v["ms"]}
            else:
                pk_, what = alu_peak(k, sm_max)
                a = v["ops"] / (v["ms"] / 1e3)
                roof_all[k] = {"bound": "alu", "achieved": a / 1e12, "peak": pk_ / 1e12, "unit": f"T{what}",
                               "frac": a / pk_, "ms": v["ms"], "peak_clock_mhz": sm_max}
        qk = build_queue(0, 1, args.instances, args.workload, args.mix)
        dom = max(pk, key=lambda k: pk[k]["ms"] * sum(1 for x in qk if x == k)) if pk else None
        roof = None
        if dom:
            # achieved inside the timed region: the dominant kind's algorithmic work over the time
            # its launches were resident (device records; co-running partners share its SMs)
            solo = roof_all[dom]
            tk = res["timed_kernels"][dom]
            w = pk[dom]
            units = w.get("ops") if solo["bound"] == "alu" else (w.get("flops") if solo["bound"] == "tensor" else w.get("bytes"))
            scale = {"alu": 1e12, "tensor": 1e12, "hbm": 1e9}[solo["bound"]]
            ach = units * tk["blocks"] / w["grid"] / (tk["busy_ms"] / 1e3) / scale
            tr = ncu_traffic(dom)
            peak_step = alu_peak(dom, sm_mhz)[0] / 1e12 if solo["bound"] == "alu" else solo["peak"]
            roof = {"bound": solo["bound"], "achieved": ach, "peak": peak_step, "unit": solo["unit"],
                    "frac": ach / peak_step,
                    **({"peak_clock_mhz": sm_mhz} if solo["bound"] == "alu" else {}), "traffic": tr["bytes_per_instance"] if tr else None,
                    "traffic_source": (f"dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set full capture "
                                       f"of the kind's whole-instance persistent launch ({tr['source']})") if tr else None,
                    "kernel": dom,
                    "measured": "timed region: algorithmic units of the kind's executed blocks / union of its "
                                "launches' resident intervals (device %globaltimer records)",
                    "solo": {"achieved": solo["achieved"], "frac": solo["frac"], "ms": solo["ms"]},
                    "units_per_instance": units}
        line = {"metric": METRIC, "value": res["value"], "unit": "kernels/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f32/bf16->f32/u32/u8 (per kernel); model f64",
                "data": "synthetic", "config": config, "clocks": res["clocks"], "gpu_launches": res["gpu_launches"],
                "e2e": res.get("e2e"), "roofline": roof,
                "speedup_vs_sequential": res["value"] / seq if seq else None,
                "speedup_vs_multistream": res["value"] / ms4 if ms4 else None,
                "baselines": bl, "roofline_all": roof_all, "device_ms_per_step": res["device_ms_per_step"],
                "phases_per_step": res["phases_per_step"], "parity": res["parity"],
                "engine_per_step": {k: res.get(k) for k in ("retunes_per_step", "stops_per_step", "memops_per_step")},
                "lease_conflicts": res["lease_conflicts"], "host_decide_ms_per_step": res["host_decide_ms_per_step"],
                "model_ms_per_step": res["model_ms_per_step"],
                "schedule_first_step": res["schedule_first_step"]}
        if not args.no_cpu and world == 1:
            try:
                line["cpu_baseline"] = cpu_oracle_leg(qk, args.size, **leg_kw)
            except Exception as e:      # never lose the GPU line to the CPU leg
                line["cpu_baseline"] = {"error": repr(e)[:300]}
        print(json.dumps(line))
        if args.json_out:
            with open(args.json_out, "w") as f:
                json.dump(line, f, indent=1)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

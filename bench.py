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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="kernelet", choices=["kernelet", "reference"])
    ap.add_argument("--instances", type=int, default=4, help="instances of each ALL-mix kernel per GPU (c2)")
    ap.add_argument("--workload", default="c2", choices=["c2", "c4", "c5"],
                    help="c2: ALL mix x4 per GPU (configs[1], default); c4: 1000 random kernels per GPU; "
                         "c5: 10,000-kernel multi-user queue over all GPUs")
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
    ap.add_argument("--levels", default="four", choices=["all", "four"],
                    help="occupancy levels per kernel (kl_config.level_mode): every b with whole warps per virtual "
                         "SM, or the four levels {1/4, 1/2, 3/4, 1} x b_max of config C2")
    ap.add_argument("--speculative", action="store_true", help="enable the speculative start (kl_config.speculative)")
    ap.add_argument("--trace-out", default=None, help="write the last timed step's launch trace (JSON lines)")
    ap.add_argument("--opt", default=None, help="OPT comparator: decide from a measured pair table "
                                               "(tools/opt_table.py) instead of the Markov model")
    return ap.parse_args()


# ---------------------------------------------------------------------------------------------
# Algorithmic work per kernel: bytes that must cross HBM, or the
# arithmetic the method must do, per instance at the given size.  Used for the roofline.
# ---------------------------------------------------------------------------------------------
def algorithmic_work(kind: str, p: dict) -> dict:
    if kind == "PC":      # one 64-B HBM3e access per random dependent load (nodes are visited
        # once: no reuse for L2) + 8 B of output per thread; ncu: 64 B DRAM read per hop
        return {"bound": "hbm", "bytes": p["n_threads"] * (p["hops"] * 64 + 8)}
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


def ncu_traffic(kind: str):
    """DRAM bytes (read + write) of one launch of `kind` from the committed `ncu --set full`
    summary (profiles/*ncu_summary.json, latest round), or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary.json")), reverse=True):
        try:
            d = json.load(open(path))
        except Exception:
            continue
        for rep, rows in d.items():
            if not isinstance(rows, list):
                continue
            for r in rows:
                if f"Body{kind}>" in r.get("kernel", "") or f"Body{kind}E" in r.get("kernel", "") or \
                        f"::Body{kind}" in r.get("kernel", ""):
                    try:
                        rd = float(str(r["dram__bytes_read.sum"]["value"]).replace(",", ""))
                        wr = float(str(r["dram__bytes_write.sum"]["value"]).replace(",", ""))
                        unit = r["dram__bytes_read.sum"]["unit"]
                        mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                        return {"bytes_per_instance": (rd + wr) * mul, "source": os.path.basename(path)}
                    except (KeyError, ValueError):
                        continue
    return None


def alu_peak(kind: str, sm_mhz: float, n_sm: int = 148) -> tuple[float, str]:
    """ALU peaks from unit counts x clock (B300_MICROARCH pipe rates): MUFU 16
    ops/clk/SM (sin, cos); SAD's VABSDIFF4 on the alu pipe, 64 lanes/clk/SM (rt 2 per SMSP);
    TEA's integer mix spreads over the alu pipe (IADD3/LOP3/SHF) and the fma pipe (IMAD), so its
    ceiling is the issue rate, 128 lanes/clk/SM."""
    f = sm_mhz * 1e6
    if kind == "MRIQ":
        return 16 * n_sm * f, "MUFU ops/s (16/clk/SM)"
    if kind == "TEA":
        return 128 * n_sm * f, "int ops/s (alu+fma pipes, issue 128/clk/SM)"
    return 64 * n_sm * f, "int ALU ops/s (64/clk/SM)"


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
def global_queue(workload: str, instances: int, world: int) -> list[str]:
    """c2 (configs[1]): ALL mix, `instances` of each kernel per GPU, round-robin arrivals.
    c4 (configs[3]): 1000 kernels per GPU drawn uniformly from ALL (seed 42).
    c5 (configs[4]): 10,000-kernel multi-user queue (16 Poisson users on CI/MI/MIX/ALL), the
    whole queue shared by all GPUs (strong scaling)."""
    if workload == "c2":
        return [e["kind"] for e in G.queue("ALL", len(ALL) * instances * world, order="round_robin")]
    if workload == "c4":
        return [e["kind"] for e in G.queue("ALL", 1000 * world, seed=42, order="uniform")]
    if workload == "c5":
        return [e["kind"] for e in G.multi_user_queue(10000, 16, seed=7)]
    raise ValueError(workload)


def build_queue(rank: int, world: int, instances: int, workload: str = "c2") -> list[str]:
    """This GPU's shard of the global queue, mix-preserving round robin."""
    from paper_1303_5164_b200.dist import shard
    return shard(global_queue(workload, instances, world), rank, world)


MODEL_FIELDS = ("rm", "r", "ipb", "pur", "mur", "m_min", "ipc_max", "pipe", "uc", "ru")


def load_profiles(path: str):
    """Calibrated model inputs (tools/calibrate.py).  Resource fields (warps, registers, shared
    memory, TMEM, b_max) are left to the runtime, which reads them from the compiled kernels."""
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        profs = {k: {f: v[f] for f in MODEL_FIELDS if f in v} for k, v in d.get("profiles", {}).items()}
        return profs, d.get("config", {})
    return None, {}


def run_kernelet(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1303_5164_b200 as K
    from paper_1303_5164_b200.workload import Instance, inputs_to_device

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    K.lib()
    kinds = build_queue(rank, world, args.instances, args.workload)
    profiles, kcfg = load_profiles(args.profile)
    t_gen = time.time()
    data = {k: G.gen(k, args.size) for k in sorted(set(kinds))}
    inputs = {k: inputs_to_device(data[k], dev) for k in data}
    # output leases: a pool of POOL output sets per kind, instance j of a kind writes set j % POOL
    # (inputs are shared read-only); the trace check below proves no two launches that were
    # resident at the same time wrote the same set
    from paper_1303_5164_b200.workload import alloc_outputs
    POOL = 4
    pools, seen, lease = {}, {}, []
    insts = []
    for k in kinds:
        j = seen.get(k, 0)
        seen[k] = j + 1
        if j < POOL:
            pools.setdefault(k, []).append(alloc_outputs(k, data[k]["params"], dev))
        insts.append(Instance(data[k], dev, inputs=inputs[k], outputs=pools[k][j % POOL]))
        lease.append((k, j % POOL))
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
    gathered = torch.zeros(world * 8, dtype=torch.int64, device=dev)

    counters[5] = rank      # kl_counters.rank / .world: the per-step reset clears fields 0-4 only
    counters[6] = world

    def one_step():
        if not args.opt:
            ctx.reset_model_cache()
        ctx.reset_counters()
        ids = ctx.submit_many([(i.kind, i.grid, i.args, n + 1, None) for n, i in enumerate(insts)])
        c = ctx.sync()
        if world > 1:
            with torch.cuda.stream(lane_a):
                dist.all_gather_into_tensor(gathered, counters)
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
    t = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    c_last = cnts[-1]
    assert c_last.kernels_done == len(insts), (c_last.kernels_done, len(insts))
    if world > 1:
        g = gathered.view(world, 8).cpu()
        assert int(g[:, 0].sum()) == len(insts) * world      # NCCL-gathered completion counters

    res = {
        "value": len(insts) * world * args.steps / (total_ms / 1e3),
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
        res["baselines"] = baselines(ctx, insts, dev, flush, barrier, args)
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


def _time_streams(fn, dev, flush, barrier, reps=3):
    import torch
    ts = []
    for _ in range(reps):
        flush.zero_()
        barrier()
        s = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn(s, e0)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def baselines(ctx, insts, dev, flush, barrier, args) -> dict:
    """Sequential (one stream, full grids at max occupancy, back to back) and plain multi-stream
    (round robin over S streams, full grids, no slicing) executions of the same kernels."""
    import torch
    out = {}

    def seq(s, e0):
        for i in insts:
            ctx.run_plain(i.kind, i.grid, i.args, s)

    ms = _time_streams(seq, dev, flush, barrier)
    out["sequential"] = {"ms_per_step": ms, "kernels_per_s": len(insts) / (ms / 1e3)}
    for S in (2, 4, 8):
        streams = [torch.cuda.Stream(device=dev) for _ in range(S)]

        def ms_fn(s, e0, streams=streams):
            evs = []
            for st in streams:
                st.wait_event(e0)
            for n, i in enumerate(insts):
                ctx.run_plain(i.kind, i.grid, i.args, streams[n % len(streams)])
            for st in streams:
                ev = torch.cuda.Event()
                ev.record(st)
                s.wait_event(ev)

        ms = _time_streams(ms_fn, dev, flush, barrier)
        out[f"multistream{S}"] = {"ms_per_step": ms, "kernels_per_s": len(insts) / (ms / 1e3)}
    return out


def per_kernel(ctx, insts, data, dev, flush, barrier) -> dict:
    """Solo plain launch of one instance of each kind: duration, algorithmic rate, roofline."""
    import torch
    out, seen = {}, set()
    for i in insts:
        if i.kind in seen:
            continue
        seen.add(i.kind)
        ms = _time_streams(lambda s, e0, i=i: ctx.run_plain(i.kind, i.grid, i.args, s), dev, flush, barrier, reps=5)
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
    """Same metric through the public API with HOST buffers: every step copies the step's inputs
    (one set per kind, shared by its instances) from pinned host memory and reads the completion
    counters back.  Each kind's copy is its kernels' arrival: the kernels are submitted with the
    copy's event as `ready_event`, so the scheduler overlaps the PCIe transfer of later kinds with
    the execution of earlier ones (arrivals trigger re-planning)."""
    import torch
    kinds_in_order = []
    for i in insts:
        if i.kind not in kinds_in_order:
            kinds_in_order.append(i.kind)
    # copy order: a two-stage flow shop (one copy stream, then the kernels), ordered by Johnson's
    # rule -- kinds whose copy is shorter than their kernel time first, by increasing copy time;
    # then the rest by decreasing kernel time -- so the last copy has the least kernel time behind
    # it (copy time from the bytes at the measured ~55 GB/s pinned H2D rate)
    if pk:
        nk = {k: sum(1 for i in insts if i.kind == k) for k in kinds_in_order}
        nbytes = {k: sum(t.numel() * t.element_size() for t in next(i for i in insts if i.kind == k).inputs.values())
                  for k in kinds_in_order}
        kinds_in_order = johnson_order(kinds_in_order, {k: nbytes[k] / 55e9 * 1e3 for k in kinds_in_order},
                                       {k: pk[k]["ms"] * nk[k] for k in kinds_in_order})
    host = {}
    for k in kinds_in_order:
        src = next(i for i in insts if i.kind == k)
        host[k] = {n: t.cpu().pin_memory() for n, t in src.inputs.items()}
    h2d = sum(t.numel() * t.element_size() for d in host.values() for t in d.values())
    copy_stream = torch.cuda.Stream(device=dev)
    ts = []
    for _ in range(max(2, min(args.steps, 3))):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(lane)
        copy_stream.wait_event(e0)
        ready = {}
        with torch.cuda.stream(copy_stream):
            for k in kinds_in_order:
                src = next(i for i in insts if i.kind == k)
                for n, t in src.inputs.items():
                    t.copy_(host[k][n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy_stream)
                ready[k] = ev
        ctx.reset_model_cache()
        ctx.reset_counters()
        ctx.submit_many([(i.kind, i.grid, i.args, n + 1, ready[i.kind]) for n, i in enumerate(insts)])
        c = ctx.sync()
        res = ctx.counters.cpu()        # D2H read of the step's result
        e1.record(lane)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
        assert int(res[0]) == len(insts)
    ms = statistics.median(ts)
    if world > 1:                       # whole-job time: the slowest rank
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": len(insts) * world / (ms / 1e3), "unit": "kernels/s", "h2d_bytes_per_step": int(h2d),
            "copy_order": kinds_in_order,
            "d2h_bytes_per_step": 64, "ms_per_step": ms, "h2d_GBps": h2d / (ms / 1e3) / 1e9}


# ---------------------------------------------------------------------------------------------
class OracleLeg:
    """The oracle as it stands, on the host cores: every kind's outputs on a fixed strided sample
    (fraction f of the elements) plus the oracle's full Alg.1 decision sequence (model + search)
    for the queue; throughput = kernels-equivalent of work done / wall time."""

    def __init__(self, kinds: list[str], size: str):
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
        self.profs = _oracle_profiles()

    def run(self, target_s: float) -> dict:
        frac = 1e-4
        t0 = time.time()
        _oracle_sample(self.O, self.data, self.sizes, frac, self.cores)
        probe = max(time.time() - t0, 1e-3)
        frac = min(1.0, frac * target_s / probe)
        t0 = time.time()
        _oracle_sample(self.O, self.data, self.sizes, frac, self.cores)
        t_k = time.time() - t0
        t0 = time.time()
        if self.profs:
            q = [{"kind": k, "blocks": 1000} for k in self.kinds]
            self.O.alg1_makespan(q, self.profs, self.O.smcfg(W=16))
        t_s = time.time() - t0
        n_equiv = frac * len(self.kinds)
        return {"value": n_equiv / (t_k + t_s), "unit": "kernels/s", "cores": self.cores, "kind": "oracle",
                "sample": f"{frac:.2e} of every output element of the {len(self.kinds)}-kernel queue (strided, "
                          f"{self.cores} threads) + the oracle's Alg.1/FindCoSchedule decision sequence; "
                          f"{t_k + t_s:.1f} s wall"}


def cpu_oracle_leg(kinds: list[str], size: str, target_s: float = 15.0) -> dict:
    return OracleLeg(kinds, size).run(target_s)


def _oracle_sample(O, data, sizes, frac, cores):
    from concurrent.futures import ThreadPoolExecutor
    jobs = []
    for k, d in data.items():
        n = sizes[k]
        m = max(1, int(n * frac))
        idx = np.linspace(0, n - 1, m).astype(np.int64)
        for chunk in np.array_split(idx, cores):
            if chunk.size:
                jobs.append((d, chunk))
    with ThreadPoolExecutor(cores) as ex:
        list(ex.map(lambda j: O.run_kernel(j[0], j[1]), jobs))


def _oracle_profiles():
    path = os.path.join(ROOT, "profiles", "kl_profile_b200.json")
    if not os.path.exists(path):
        return None
    d = json.load(open(path))["profiles"]
    return {k: v for k, v in d.items() if k in ALL}


# ---------------------------------------------------------------------------------------------
def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    n_global = len(global_queue(args.workload, args.instances, world))
    wl_name = {"c2": f"ALL mix x{args.instances} per GPU ({len(ALL) * args.instances} kernels, {args.size} sizes, "
                     "all pending at t=0)",
               "c4": f"1000 kernels per GPU uniform over ALL (seed 42), {args.size} sizes",
               "c5": f"10,000-kernel multi-user queue (16 Poisson users, CI/MI/MIX/ALL), {args.size} sizes"}[args.workload]
    config = {"workload": wl_name, "global_kernels": n_global,
              "sizes": "tb:description (million = 2^20), MRIQ numK = 2048", "parallelism": f"queue shard x{world}",
              "l2": "256 MiB write between steps; inputs >> L2", "model_cache": "cleared every step",
              "split_rule": "argmax CP over (pair, ratio)" if args.split_rule == 1 else "argmin dT (Eq.8)",
              "cp_min": args.cp_min or 0.0, "decisions_from": "measured pair table (OPT)" if args.opt else "Markov model",
              "occupancy_levels": "{1/4, 1/2, 3/4, 1} x b_max per kernel (config C2)" if args.levels == "four"
              else "every b with whole warps per virtual SM"}

    if args.impl == "reference":
        if rank != 0:
            return
        kinds = build_queue(0, 1, args.instances, args.workload)
        leg = OracleLeg(kinds, args.size)
        vals = []
        for s in range(args.warmup + args.steps):
            r = leg.run(target_s=max(2.0, 60.0 / (args.warmup + args.steps)))
            if s >= args.warmup:
                vals.append(r["value"])
        v = statistics.median(vals)
        line = {"metric": METRIC, "value": v, "unit": "kernels/s", "impl": "reference", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong" if args.workload == "c5" else "weak",
                "vs_baseline": None, "dtype": "f32/f64/u32 (per kernel)", "data": "synthetic", "config": config,
                "cpu_baseline": {**r, "value": v}, "e2e": {"value": v, "unit": "kernels/s", "h2d_bytes_per_step": 0,
                                                          "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_kernelet(args, rank, world, local_rank)
    if rank == 0:
        bl = res.get("baselines", {})
        seq = bl.get("sequential", {}).get("kernels_per_s")
        ms4 = max((v["kernels_per_s"] for k, v in bl.items() if k.startswith("multistream")), default=None)
        pk = res.get("per_kernel", {})
        sm_mhz = (res["clocks"].get("sm_mhz") or 1965.0)
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
                pk_, what = alu_peak(k, sm_mhz)
                a = v["ops"] / (v["ms"] / 1e3)
                roof_all[k] = {"bound": "alu", "achieved": a / 1e12, "peak": pk_ / 1e12, "unit": f"T{what}",
                               "frac": a / pk_, "ms": v["ms"]}
        qk = build_queue(0, 1, args.instances, args.workload)
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
            roof = {"bound": solo["bound"], "achieved": ach, "peak": solo["peak"], "unit": solo["unit"],
                    "frac": ach / solo["peak"], "traffic": tr["bytes_per_instance"] if tr else None,
                    "traffic_source": (f"dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set full capture "
                                       f"of the kind's whole-instance persistent launch ({tr['source']})") if tr else None,
                    "kernel": dom,
                    "measured": "timed region: algorithmic units of the kind's executed blocks / union of its "
                                "launches' resident intervals (device %globaltimer records)",
                    "solo": {"achieved": solo["achieved"], "frac": solo["frac"], "ms": solo["ms"]},
                    "units_per_instance": units}
        line = {"metric": METRIC, "value": res["value"], "unit": "kernels/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
                "scaling": "strong" if args.workload == "c5" else "weak", "vs_baseline": None, "dtype": "f32/bf16->f32/u32/u8 (per kernel); model f64",
                "data": "synthetic", "config": config, "clocks": res["clocks"], "gpu_launches": res["gpu_launches"],
                "e2e": res.get("e2e"), "roofline": roof,
                "speedup_vs_sequential": res["value"] / world / seq if seq else None,
                "speedup_vs_multistream": res["value"] / world / ms4 if ms4 else None,
                "baselines": bl, "roofline_all": roof_all, "device_ms_per_step": res["device_ms_per_step"],
                "phases_per_step": res["phases_per_step"], "parity": res["parity"],
                "engine_per_step": {k: res.get(k) for k in ("retunes_per_step", "stops_per_step", "memops_per_step")},
                "lease_conflicts": res["lease_conflicts"], "host_decide_ms_per_step": res["host_decide_ms_per_step"],
                "model_ms_per_step": res["model_ms_per_step"],
                "schedule_first_step": res["schedule_first_step"]}
        if not args.no_cpu and world == 1:
            try:
                line["cpu_baseline"] = cpu_oracle_leg(build_queue(0, 1, args.instances, args.workload), args.size)
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

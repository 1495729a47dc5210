"""A/B of the MRIQ MUFU/polynomial mix (KL_MRIQ_G, KL_MRIQ_P): build one libkl.so per variant
(`build`, CPU) and time each on the GPU (`run`): solo plain-grid device time at paper size (L2
flushed, median of 7); parity of a variant build is tests/test_gpu_kernels.py (tools/ never
imports oracle/)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANTS = [(16, 0), (16, 1), (8, 1), (8, 2), (4, 1), (12, 1), (12, 2)]


def lib(g, p):
    return os.path.join(ROOT, "variants", f"libkl_mriq_{g}_{p}.so")


def build():
    sys.path.insert(0, ROOT)
    import paper_1303_5164_b200 as K
    os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
    procs = []
    for g, p in VARIANTS:
        cmd = (["nvcc"] + K.NVCC_FLAGS + [f"-DKL_MRIQ_G={g}", f"-DKL_MRIQ_P={p}", "-o", lib(g, p)]
               + [os.path.join(ROOT, "paper_1303_5164_b200", s) for s in K.SOURCES])
        procs.append(subprocess.Popen(cmd, cwd=os.path.join(ROOT, "paper_1303_5164_b200")))
    assert all(pr.wait() == 0 for pr in procs)


def one():
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import kl_inputs as G
    import paper_1303_5164_b200 as K
    from paper_1303_5164_b200.workload import Instance
    ctx = K.Context(device=0)
    err = None      # parity of the variant: tests/test_gpu_kernels.py on the variant build
    i = Instance(G.gen("MRIQ", "paper"), "cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    ts = []
    for _ in range(7):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.run_plain("MRIQ", i.grid, i.args, 0)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    pers = sorted(ctx.run_capped("MRIQ", i.grid, i.args, 0) for _ in range(7))[3]
    print(json.dumps({"ms": sorted(ts)[3], "persistent_ms": pers, "err": err}))


def run():
    out = {}
    for g, p in VARIANTS:
        env = dict(os.environ, KL_LIB_PATH=lib(g, p))
        r = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True)
        res = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {"error": r.stderr[-500:]}
        out[f"G{g}P{p}"] = res
        print(f"G={g:2d} P={p}  f={p / g:.3f}  {res}", flush=True)
    return out


if __name__ == "__main__":
    {"build": build, "run": run, "one": one}[sys.argv[1]]()

"""A/B builds of libkl.so with compile-time knobs (-D...), CPU side: `build NAME=-DA=1,-DB=2 ...`
writes variants/libkl_NAME.so; GPU side: `run CMD NAME...` runs CMD once per variant with
KL_LIB_PATH pointing at it (e.g. CMD = "python tools/launcher_overhead.py")."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def lib(name):
    return os.path.join(ROOT, "variants", f"libkl_{name}.so")


def build(specs):
    sys.path.insert(0, ROOT)
    import paper_1303_5164_b200 as K
    os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
    procs = []
    for spec in specs:
        name, _, defs = spec.partition("=")
        cmd = (["nvcc"] + K.NVCC_FLAGS + [d for d in defs.split(",") if d] + ["-o", lib(name)]
               + [os.path.join(ROOT, "paper_1303_5164_b200", s) for s in K.SOURCES])
        procs.append(subprocess.Popen(cmd, cwd=os.path.join(ROOT, "paper_1303_5164_b200")))
    assert all(p.wait() == 0 for p in procs)


def run(cmd, names):
    for name in names:
        print(f"== {name}", flush=True)
        subprocess.run(cmd, shell=True, env=dict(os.environ, KL_LIB_PATH=lib(name)))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        run(sys.argv[2], sys.argv[3:])

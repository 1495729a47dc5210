"""Device-memory plumbing: turn kl_inputs instances into torch tensors + kl_args structs.

Only allocation, host<->device copies and pointer marshalling live here; every arithmetic step
runs in libkl.so.  Output buffers can be leased from a pool so co-scheduled instances never
alias a written buffer (SURVEY §4 race detection: buffer leases)."""
from __future__ import annotations

import numpy as np
import torch

from . import ARGS, KIND_ID

_NP2T = {np.float32: torch.float32, np.int32: torch.int32, np.uint32: torch.int32,
         np.uint16: torch.int16, np.uint8: torch.uint8, np.int64: torch.int64}

OUTPUTS = {  # name -> (numpy dtype, element count from params)
    "PC": lambda p: {"out": (np.int32, p["n_threads"]), "acc": (np.uint32, p["n_threads"])},
    "SAD": lambda p: {"sad": (np.uint16, (p["width"] // 16) * (p["height"] // 16) * 1089)},
    "SPMV": lambda p: {"y": (np.float32, p["n_rows"])},
    "ST": lambda p: {"out": (np.float32, p["nx"] * p["ny"] * p["nz"])},
    "MM": lambda p: {"C": (np.float32, p["M"] * p["N"])},
    "MRIQ": lambda p: {"qr": (np.float32, p["num_x"]), "qi": (np.float32, p["num_x"])},
    "BS": lambda p: {"call": (np.float32, p["n"]), "put": (np.float32, p["n"])},
    "TEA": lambda p: {"out": (np.uint32, 2 * p["n"])},
    "MATADD": lambda p: {"C": (np.float32, p["n"] * p["n"])},
    "SYNTH": lambda p: {"y": (np.float32, p["n"])},
}
INPUTS = {
    "PC": ["next"], "SAD": ["cur", "ref"], "SPMV": ["rowptr", "cols", "vals", "x"], "ST": ["inp"],
    "MM": ["A", "Bt"], "MRIQ": ["x", "y", "z", "kx", "ky", "kz", "phimag"], "BS": ["S", "X", "T"],
    "TEA": ["v"], "MATADD": ["A", "B"], "SYNTH": ["x"],
}


def to_device(a: np.ndarray, device, pin: bool = False) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    t = torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else
                         a.view(np.int32) if a.dtype == np.uint32 else a)
    if device == "cpu":
        return t.pin_memory() if pin else t
    return t.to(device, non_blocking=False)


def alloc_outputs(kind: str, p: dict, device) -> dict:
    return {n: torch.empty(cnt, dtype=_NP2T[dt], device=device) for n, (dt, cnt) in OUTPUTS[kind](p).items()}


def inputs_to_device(d: dict, device) -> dict:
    return {n: to_device(d[n], device) for n in INPUTS[d["kind"]]}


def make_args(kind: str, p: dict, inp: dict, out: dict, **over):
    A = ARGS[KIND_ID[kind]]
    ptr = lambda t: t.data_ptr()
    if kind == "PC":
        return A(ptr(inp["next"]), ptr(out["out"]), ptr(out["acc"]), p["n_nodes"], p["hops"], p["n_threads"])
    if kind == "SAD":
        return A(ptr(inp["cur"]), ptr(inp["ref"]), ptr(out["sad"]), p["width"], p["height"])
    if kind == "SPMV":
        return A(ptr(inp["rowptr"]), ptr(inp["cols"]), ptr(inp["vals"]), ptr(inp["x"]), ptr(out["y"]), p["n_rows"])
    if kind == "ST":
        c0 = over.get("c0", p.get("c0", 1.0 / 6.0))
        c1 = over.get("c1", p.get("c1", 1.0 / 36.0))
        return A(ptr(inp["inp"]), ptr(out["out"]), p["nx"], p["ny"], p["nz"], c0, c1)
    if kind == "MM":
        return A(ptr(inp["A"]), ptr(inp["Bt"]), ptr(out["C"]), p["M"], p["N"], p["K"])
    if kind == "MRIQ":
        return A(*(ptr(inp[n]) for n in INPUTS["MRIQ"]), ptr(out["qr"]), ptr(out["qi"]), p["num_x"], p["num_k"])
    if kind == "BS":
        return A(ptr(inp["S"]), ptr(inp["X"]), ptr(inp["T"]), ptr(out["call"]), ptr(out["put"]), p["n"],
                 p.get("R", 0.02), p.get("V", 0.30))
    if kind == "TEA":
        a = A(ptr(inp["v"]), ptr(out["out"]), p["n"])
        for i in range(4):
            a.key[i] = int(p["key"][i])
        return a
    if kind == "MATADD":
        return A(ptr(inp["A"]), ptr(inp["B"]), ptr(out["C"]), p["n"])
    if kind == "SYNTH":
        return A(ptr(inp["x"]), ptr(out["y"]), p["n"], p["fmas"], p.get("a", 0.999), p.get("b", 0.001))
    raise KeyError(kind)


class Instance:
    """One kernel instance: device inputs (possibly shared), leased outputs, kl_args struct."""

    def __init__(self, d: dict, device, inputs: dict | None = None, outputs: dict | None = None, **over):
        self.kind = d["kind"]
        self.params = dict(d["params"])
        if self.kind == "TEA":
            self.params["key"] = [int(x) for x in d["key"]]
        self.grid = d["grid_blocks"]
        self.inputs = inputs if inputs is not None else inputs_to_device(d, device)
        self.outputs = outputs if outputs is not None else alloc_outputs(self.kind, self.params, device)
        self.args = make_args(self.kind, self.params, self.inputs, self.outputs, **over)

    def result(self) -> dict:
        """Outputs as numpy arrays with the oracle's names and dtypes."""
        res = {}
        for n, (dt, _) in OUTPUTS[self.kind](self.params).items():
            res[n] = self.outputs[n].cpu().numpy().view(dt)
        return res

    def input_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.inputs.values())

    def output_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.outputs.values())

#!/usr/bin/env python
"""cuBLAS bf16 GEMM (torch.matmul) on MM's shapes: what the library reaches on this box (context
for MM's roofline; never on the product path).  usage: python tools/cublas_ref.py"""
import statistics
import sys

import torch

shapes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1:]] or [(8192, 2048, 2048), (8192, 2048, 4096),
                                                                         (2048, 2048, 2048), (8192, 8192, 8192)]
for M, N, K in shapes:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    for out_dtype in (torch.bfloat16, torch.float32):
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            c = torch.matmul(a, b.t()) if out_dtype == torch.bfloat16 else torch.mm(a.float(), b.float().t()) if False else torch.matmul(a, b.t()).float()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts[3:])
        print(f"cuBLAS {M}x{N}x{K} ({'bf16 out' if out_dtype == torch.bfloat16 else 'bf16 out + cast'}): "
              f"{ms * 1e3:.1f} us, {2 * M * N * K / ms / 1e9:.0f} TF/s", flush=True)

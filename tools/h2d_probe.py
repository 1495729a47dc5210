import torch, time
n = 1 << 28  # 1 GiB float32 = 4 bytes * 2^28
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for ns in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    chunk = n // ns
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i*chunk:(i+1)*chunk].copy_(h[i*chunk:(i+1)*chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(ns, "streams", round(4 * n / dt / 1e9, 1), "GB/s")

# Raw pinned host<->device bandwidth on the box (the e2e bound): python tools/pcie_bw.py
import torch, time
n = 705 * 1024 * 1024 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
o = torch.empty(252 * 1024 * 1024 // 8, dtype=torch.float64).pin_memory()
do = torch.empty_like(o, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter() - t
    t = time.perf_counter(); o.copy_(do, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): o.copy_(do, non_blocking=True)
    torch.cuda.synchronize(); t3 = time.perf_counter() - t
    print("H2D %.1f GB/s  D2H %.1f GB/s  both-overlapped %.2f ms (H2D-only %.2f ms)" % (h.numel() * 8 / t1 / 1e9, o.numel() * 8 / t2 / 1e9, t3 * 1e3, t1 * 1e3))

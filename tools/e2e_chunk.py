#!/usr/bin/env python3
"""End-to-end host-API time (vd_batch_forward_dynamics_host, pinned fp64 host
buffers, Panda 4M states: 705 MB in, 252 MB out) against the pipeline chunk
size (internal knob vdi_set_host_chunk_bytes; the last two chunks' worth
is split into halving chunks), next to the raw pinned copy
rates of the same box.

Usage: python tools/e2e_chunk.py [N]
"""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_04310_b200 as vd  # noqa: E402
from paper_2604_04310_b200 import _lib  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 4194304
    lib = _lib.load()
    lib.vdi_set_host_chunk_bytes.argtypes = [ctypes.c_int64]
    lib.vdi_set_host_chunk_bytes.restype = None
    m = vd.robots.chain7()
    n = m.dof()
    g = torch.Generator().manual_seed(1)
    hq, hqd, htau = [((torch.rand((n, N), generator=g, dtype=torch.float64) * 2 - 1) * 3.14).pin_memory()
                     for _ in range(3)]
    hout = torch.empty((n, N), dtype=torch.float64).pin_memory()
    hst = torch.empty(N, dtype=torch.int32).pin_memory()
    devs = (ctypes.c_int * 1)(0)
    torch.cuda.init()

    def step():
        rc = lib.vd_batch_forward_dynamics_host(m.handle, N, hq.data_ptr(), hqd.data_ptr(), htau.data_ptr(), None,
                                                hout.data_ptr(), hst.data_ptr(), devs, 1)
        assert rc == 0, lib.vd_last_error().decode()

    moved = (3 * n * N + n * N) * 8 + 4 * N
    for mb in (24, 48, 96, 192):
        lib.vdi_set_host_chunk_bytes(mb << 20)
        step()
        ts = []
        for _ in range(5):
            t = time.perf_counter()
            step()
            ts.append(time.perf_counter() - t)
        best, med = min(ts), sorted(ts)[2]
        print(f"chunk {mb:4d} MB  median {med * 1e3:7.2f} ms  best {best * 1e3:7.2f} ms  "
              f"{N / med:.3e} evals/s  {moved / med / 1e9:5.1f} GB/s", flush=True)
    lib.vdi_set_host_chunk_bytes(0)
    # raw pinned copies of the same byte counts
    d_in = torch.empty((3, n, N), dtype=torch.float64, device="cuda")
    d_out = torch.empty((n, N), dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for k, h in enumerate((hq, hqd, htau)):
            d_in[k].copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter() - t
        t = time.perf_counter()
        hout.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter() - t
        t = time.perf_counter()
        with torch.cuda.stream(s1):
            for k, h in enumerate((hq, hqd, htau)):
                d_in[k].copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize()
        t3 = time.perf_counter() - t
        print(f"raw: H2D {3 * n * N * 8 / t1 / 1e9:.1f} GB/s ({t1 * 1e3:.2f} ms), D2H {n * N * 8 / t2 / 1e9:.1f} GB/s "
              f"({t2 * 1e3:.2f} ms), both overlapped {t3 * 1e3:.2f} ms", flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Bandwidth of vd_rows_to_planes / vd_planes_to_rows against torch's
strided copy (.t().contiguous()).  Usage: python tools/layout_time.py"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_04310_b200 as vd  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    lib = vd._lib.load()
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    for K, N in ((7, 4194304), (29, 4194304), (42, 4194304), (174, 1048576)):
        for dt, code in ((torch.float64, 0), (torch.float32, 1)):
            x = torch.rand((N, K), device="cuda", dtype=torch.float64).to(dt)
            y = torch.empty((K, N), device="cuda", dtype=dt)
            gb = 2 * x.numel() * x.element_size() / 1e6  # MB -> GB/s with ms
            t_torch = timeit(lambda: x.t().contiguous())
            t_r2p = timeit(lambda: lib.vd_rows_to_planes(code, N, K, p(x), K, p(y), N, None))
            t_p2r = timeit(lambda: lib.vd_planes_to_rows(code, N, K, p(y), N, p(x), K, None))
            print(f"K={K:3d} N={N} {str(dt)[6:]:8s} torch {gb / t_torch:7.0f} GB/s  rows->planes {gb / t_r2p:7.0f} GB/s"
                  f"  planes->rows {gb / t_p2r:7.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()

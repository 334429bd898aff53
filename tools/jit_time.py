#!/usr/bin/env python3
"""Per-model JIT modules against the loop kernels, device-timed through the
C-ABI on plane-layout buffers.  Usage: python tools/jit_time.py [N]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2604_04310_b200 as vd  # noqa: E402
from urdf_gen import random_urdf  # noqa: E402


def timeit(fn, reps=10):
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
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
    lib = vd._lib.load()
    for name, m in (("humanoid23", vd.robots.by_name("humanoid23")),
                    ("random16", vd.urdf.load_model_from_string(random_urdf(11, n=16, branchiness=0.6)))):
        n = m.dof()
        dj = vd.DeviceModel(m, 0, jit=True)
        dg = vd.DeviceModel(m, 0, generic=True)
        for dt, code in ((torch.float64, 0), (torch.float32, 1)):
            x = [((torch.rand((n, N), device="cuda", dtype=torch.float64) * 2 - 1) * np.pi).to(dt) for _ in range(3)]
            out = torch.empty((n * n, N), dtype=dt, device="cuda")
            st = torch.empty(N, dtype=torch.int32, device="cuda")
            p = [t.data_ptr() for t in x]
            for dm, mode in ((dg, "loop"), (dj, "jit")):
                h = dm.handle
                ops = {"rnea": lambda: lib.vd_rnea(h, code, N, p[0], p[1], p[2], N, None, None, out.data_ptr(), N, None),
                       "crba": lambda: lib.vd_crba(h, code, N, p[0], N, out.data_ptr(), N, None),
                       "aba": lambda: lib.vd_aba(h, code, N, p[0], p[1], p[2], N, None, None, out.data_ptr(), N,
                                                 st.data_ptr(), None),
                       "fk": lambda: lib.vd_fk(h, code, N, p[0], N, out.data_ptr(), N, None)}
                if 12 * n > n * n:
                    ops.pop("fk")
                for op, fn in ops.items():
                    assert fn() == 0, lib.vd_last_error()
                    print(f"{name} n={n} {str(dt)[6:]} {op:5s} {mode:4s} {timeit(fn):.4f} ms", flush=True)


if __name__ == "__main__":
    main()

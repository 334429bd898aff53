#!/usr/bin/env python3
"""Device-timed RNEA / bias / forward dynamics with one gravity per call
against per-state gravity (vd_*_pg), through the C-ABI on plane-layout
buffers; generated kernels (chain7, tree29) and the loop kernels (humanoid23).
Usage: gravity_time.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_04310_b200 as vd  # noqa: E402
from fext_time import timeit  # noqa: E402


def main():
    lib = vd._lib.load()
    for robot, N in (("chain7", 4194304), ("tree29", 262144), ("humanoid23", 262144)):
        m = vd.robots.by_name(robot)
        dm = vd.DeviceModel(m, 0)
        n = m.dof()
        for dt in (torch.float64, torch.float32):
            code = 0 if dt == torch.float64 else 1
            P = [((torch.rand((n, N), device="cuda", dtype=torch.float64) * 2 - 1) * np.pi).to(dt) for _ in range(3)]
            G = (torch.rand((3, N), device="cuda", dtype=torch.float64) * 20 - 10).to(dt)
            out = torch.empty((n, N), dtype=dt, device="cuda")
            st = torch.empty(N, dtype=torch.int32, device="cuda")
            p = [t.data_ptr() for t in P]
            calls = {
                "rnea": lambda: lib.vd_rnea(dm.handle, code, N, p[0], p[1], p[2], N, None, None, out.data_ptr(), N,
                                            None),
                "rnea_pg": lambda: lib.vd_rnea_pg(dm.handle, code, N, p[0], p[1], p[2], N, G.data_ptr(), None,
                                                  out.data_ptr(), N, None),
                "bias": lambda: lib.vd_bias(dm.handle, code, N, p[0], p[1], N, None, None, out.data_ptr(), N, None),
                "bias_pg": lambda: lib.vd_bias_pg(dm.handle, code, N, p[0], p[1], N, G.data_ptr(), None,
                                                  out.data_ptr(), N, None),
                "aba": lambda: lib.vd_aba(dm.handle, code, N, p[0], p[1], p[2], N, None, None, out.data_ptr(), N,
                                          st.data_ptr(), None),
                "aba_pg": lambda: lib.vd_aba_pg(dm.handle, code, N, p[0], p[1], p[2], N, G.data_ptr(), None,
                                                out.data_ptr(), N, st.data_ptr(), None),
            }
            for nm, fn in calls.items():
                assert fn() == 0, lib.vd_last_error()
                print(robot, N, str(dt)[6:], nm, round(timeit(fn), 4), "ms", flush=True)


if __name__ == "__main__":
    main()

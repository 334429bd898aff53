#!/usr/bin/env python3
"""Per-model JIT modules against the loop kernels, device-timed through the
C-ABI on plane-layout buffers.  Usage: python tools/jit_time.py [N]"""
import ctypes
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
        frame = "l_palm" if name == "humanoid23" else "tool"
        dj = vd.DeviceModel(m, 0, jit=True, jit_frames=(frame,))
        dg = vd.DeviceModel(m, 0, generic=True)
        for dt, code in ((torch.float64, 0), (torch.float32, 1)):
            x = [((torch.rand((n, N), device="cuda", dtype=torch.float64) * 2 - 1) * np.pi).to(dt) for _ in range(3)]
            out = torch.empty((max(n * n, 12 + 6 * n, 36), N), dtype=dt, device="cuda")
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
                P = vd._lib.OscParams()
                P.frame = m.frame_index(frame)
                for k in range(9):
                    P.target[k] = 1.0 if k in (0, 4, 8) else 0.0
                for k in range(6):
                    P.kp[k], P.kd[k] = 100.0, 20.0
                post = (ctypes.c_double * n)(*([0.0] * n))
                P.posture = ctypes.cast(post, vd._lib.Pd)
                P.posture_kp, P.posture_kd, P.epsilon = 10.0, 2.0, 1e-6
                P.gravity[2] = 9.81
                lam = out[:36]
                ops["osc"] = lambda: lib.vd_osc(h, code, N, p[0], p[1], N, ctypes.byref(P), out.data_ptr(),
                                                lam.data_ptr(), N, st.data_ptr(), None)
                ops["jac"] = lambda: lib.vd_jacobian(h, code, N, p[0], N, P.frame, out.data_ptr(),
                                                     out[12:].data_ptr(), N, None)
                for op, fn in ops.items():
                    assert fn() == 0, lib.vd_last_error()
                    print(f"{name} n={n} {str(dt)[6:]} {op:5s} {mode:4s} {timeit(fn):.4f} ms", flush=True)


if __name__ == "__main__":
    main()

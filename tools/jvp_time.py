#!/usr/bin/env python3
"""A/B timing of the forward-mode JVP kernels through the Python API.

Usage: python tools/jvp_time.py [robot] [N]   (default tree29 262144)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_04310_b200 as vd  # noqa: E402


def main():
    robot = sys.argv[1] if len(sys.argv) > 1 else "tree29"
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
    m = vd.robots.by_name(robot)
    dm = vd.DeviceModel(m, 0)
    n = m.dof()
    for dt in (torch.float64, torch.float32):
        g = torch.Generator(device="cuda").manual_seed(1)
        X = [((torch.rand((N, n), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) * 3.14159).to(dt)
             for _ in range(6)]
        fns = {"fk_jvp": lambda: vd.forward_kinematics_jvp(dm, X[0], X[1]),
               "rnea_jvp": lambda: vd.rnea_jvp(dm, X[0], X[1], X[2], X[3], X[4], X[5]),
               "crba_jvp": lambda: vd.crba_jvp(dm, X[0], X[1]),
               "aba_jvp": lambda: vd.forward_dynamics_jvp(dm, X[0], X[1], X[2], X[3], X[4], X[5])}
        for k, f in fns.items():
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                f()
            b.record()
            torch.cuda.synchronize()
            print(robot, N, str(dt)[6:], k, round(a.elapsed_time(b) / 10, 4), "ms", flush=True)
        # the C-ABI call alone on plane-layout (SoA) buffers: no layout conversion
        import ctypes
        from paper_2604_04310_b200 import _lib
        lib = _lib.load()
        P = [x.T.contiguous() for x in X]
        out = torch.empty_like(P[0])
        dout = torch.empty_like(P[0])
        g3 = (ctypes.c_double * 3)(0.0, 0.0, 9.81)
        st = torch.empty(N, dtype=torch.int32, device="cuda")
        dti = 0 if dt == torch.float64 else 1
        s = torch.cuda.current_stream().cuda_stream

        def abi():
            rc = lib.vd_aba_jvp(dm.handle, dti, N, P[0].data_ptr(), P[1].data_ptr(), P[2].data_ptr(), P[3].data_ptr(),
                                P[4].data_ptr(), P[5].data_ptr(), N, g3, None, out.data_ptr(), dout.data_ptr(), N,
                                st.data_ptr(), s)
            assert rc == 0, lib.vd_last_error().decode()
        for _ in range(3):
            abi()
        torch.cuda.synchronize()
        a.record()
        for _ in range(10):
            abi()
        b.record()
        torch.cuda.synchronize()
        print(robot, N, str(dt)[6:], "vd_aba_jvp (C-ABI, planes)", round(a.elapsed_time(b) / 10, 4), "ms", flush=True)


if __name__ == "__main__":
    main()

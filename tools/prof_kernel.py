#!/usr/bin/env python3
"""Minimal driver for ncu captures: a few launches of one hot-path kernel.

Usage: python tools/prof_kernel.py [aba|rnea|crba|crbap|dyn|osc|fk] [chain7|tree29] [f64|f32] [N] [launches]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_04310_b200 as vd  # noqa: E402


def main():
    op = sys.argv[1] if len(sys.argv) > 1 else "aba"
    robot = sys.argv[2] if len(sys.argv) > 2 else "chain7"
    dt = sys.argv[3] if len(sys.argv) > 3 else "f64"
    N = int(sys.argv[4]) if len(sys.argv) > 4 else 4194304
    launches = int(sys.argv[5]) if len(sys.argv) > 5 else 4
    code = 0 if dt == "f64" else 1
    tdt = torch.float64 if dt == "f64" else torch.float32
    m = vd.robots.by_name(robot)
    dm = vd.DeviceModel(m, 0)
    n = m.dof()
    g = torch.Generator(device="cuda").manual_seed(1)
    x = [((torch.rand((n, N), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) * np.pi).to(tdt)
         for _ in range(3)]
    out = torch.empty((max(n * n, 12 * n), N), dtype=tdt, device="cuda")
    lib = vd._lib.load()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(launches):
        if op == "aba":
            rc = lib.vd_aba(dm.handle, code, N, x[0].data_ptr(), x[1].data_ptr(), x[2].data_ptr(), N, None, None,
                            out.data_ptr(), N, None, s)
        elif op == "rnea":
            rc = lib.vd_rnea(dm.handle, code, N, x[0].data_ptr(), x[1].data_ptr(), x[2].data_ptr(), N, None, None,
                             out.data_ptr(), N, s)
        elif op == "crba":
            rc = lib.vd_crba(dm.handle, code, N, x[0].data_ptr(), N, out.data_ptr(), N, s)
        elif op == "crbap":
            rc = lib.vd_crba_packed(dm.handle, code, N, x[0].data_ptr(), N, out.data_ptr(), N, s)
        elif op == "dyn":  # vd_dynamics: M (n² planes), bias, q̈
            if _ == 0:
                bq = torch.empty((n, N), dtype=tdt, device="cuda")
                aq = torch.empty((n, N), dtype=tdt, device="cuda")
            rc = lib.vd_dynamics(dm.handle, code, N, x[0].data_ptr(), x[1].data_ptr(), x[2].data_ptr(), N, None,
                                 out.data_ptr(), bq.data_ptr(), aq.data_ptr(), N, None, s)
        elif op == "fk":
            rc = lib.vd_fk(dm.handle, code, N, x[0].data_ptr(), N, out.data_ptr(), N, s)
        elif op == "osc":
            if _ == 0:
                frame = "ee" if robot == "chain7" else "l_palm"
                P = vd._lib.OscParams()
                P.frame = m.frame_index(frame)
                pose = vd.frame_transform(dm, torch.zeros((1, n), dtype=torch.float64, device="cuda"), frame)
                pose = pose.cpu().numpy()[0]
                for k in range(12):
                    P.target[k] = float(pose[k])
                for k in range(6):
                    P.kp[k], P.kd[k], P.accel_ff[k] = 100.0, 20.0, 0.0
                post = (ctypes.c_double * n)(*([0.0] * n))
                P.posture = ctypes.cast(post, vd._lib.Pd)
                P.posture_kp, P.posture_kd, P.epsilon = 10.0, 2.0, 1e-6
                P.gravity[0], P.gravity[1], P.gravity[2] = 0.0, 0.0, 9.81
                lam = torch.empty((36, N), dtype=tdt, device="cuda")
            rc = lib.vd_osc(dm.handle, code, N, x[0].data_ptr(), x[1].data_ptr(), N, ctypes.byref(P), out.data_ptr(),
                            lam.data_ptr(), N, None, s)
        else:
            raise SystemExit("unknown op " + op)
        assert rc == 0, lib.vd_last_error()
    torch.cuda.synchronize()
    print("ok", op, robot, dt, N, launches)


if __name__ == "__main__":
    main()

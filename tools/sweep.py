#!/usr/bin/env python3
"""Device-timed sweep of every kernel × robot × dtype × (specialised | generic).

Usage: python tools/sweep.py [--n-chain 4194304] [--n-tree 262144] [--ops aba,rnea,...]
Prints one JSON object per line (robot, op, dtype, mode, N, ms, evals/s).
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_04310_b200 as vd  # noqa: E402


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-chain", type=int, default=4194304)
    ap.add_argument("--n-tree", type=int, default=262144)
    ap.add_argument("--ops", default="fk,jac,rnea,crba,aba,dyn,osc")
    ap.add_argument("--robots", default="chain7,tree29")
    ap.add_argument("--dtypes", default="f64,f32")
    ap.add_argument("--modes", default="spec,generic")
    a = ap.parse_args()
    lib = vd._lib.load()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for robot in a.robots.split(","):
        m = vd.robots.by_name(robot)
        n = m.dof()
        N = a.n_chain if robot == "chain7" else a.n_tree
        frame = m.frame_index("ee" if robot == "chain7" else "l_palm")
        for dt in a.dtypes.split(","):
            code = 0 if dt == "f64" else 1
            tdt = torch.float64 if dt == "f64" else torch.float32
            g = torch.Generator(device="cuda").manual_seed(3)
            x = [((torch.rand((n, N), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) * np.pi).to(tdt)
                 for _ in range(3)]
            out = torch.empty((max(n * n, 12 * n), N), dtype=tdt, device="cuda")
            o2 = torch.empty((n, N), dtype=tdt, device="cuda")
            o3 = torch.empty((36, N), dtype=tdt, device="cuda")
            P = vd._lib.OscParams()
            P.frame = frame
            for k in range(9):
                P.target[k] = 1.0 if k in (0, 4, 8) else 0.0
            for k in range(6):
                P.kp[k], P.kd[k] = 100.0, 20.0
            post = (ctypes.c_double * n)(*([0.0] * n))
            P.posture = ctypes.cast(post, vd._lib.Pd)
            P.posture_kp, P.posture_kd, P.epsilon = 10.0, 2.0, 1e-6
            P.gravity[2] = 9.81
            for mode in a.modes.split(","):
                dm = vd.DeviceModel(m, 0, generic=(mode == "generic"))
                h = dm.handle
                p = [t.data_ptr() for t in x]
                calls = {
                    "fk": lambda: lib.vd_fk(h, code, N, p[0], N, out.data_ptr(), N, s),
                    "jac": lambda: lib.vd_jacobian(h, code, N, p[0], N, frame, o3.data_ptr(), out.data_ptr(), N, s),
                    "rnea": lambda: lib.vd_rnea(h, code, N, p[0], p[1], p[2], N, None, None, o2.data_ptr(), N, s),
                    "crba": lambda: lib.vd_crba(h, code, N, p[0], N, out.data_ptr(), N, s),
                    "aba": lambda: lib.vd_aba(h, code, N, p[0], p[1], p[2], N, None, None, o2.data_ptr(), N, None, s),
                    "dyn": lambda: lib.vd_dynamics(h, code, N, p[0], p[1], p[2], N, None, out.data_ptr(),
                                                   o3.data_ptr(), o2.data_ptr(), N, None, s),
                    "osc": lambda: lib.vd_osc(h, code, N, p[0], p[1], N, ctypes.byref(P), o2.data_ptr(),
                                              o3.data_ptr(), N, None, s),
                }
                for op in a.ops.split(","):
                    rc = calls[op]()
                    if rc:
                        print(json.dumps({"robot": robot, "op": op, "dtype": dt, "mode": mode, "error": rc}))
                        continue
                    ms = timeit(calls[op], reps=10 if N * n > 4e7 else 20)
                    print(json.dumps({"robot": robot, "op": op, "dtype": dt, "mode": mode, "N": N, "ms": round(ms, 4),
                                      "evals_per_s": round(N / (ms * 1e-3))}), flush=True)
            del x, out, o2, o3
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

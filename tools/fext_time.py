#!/usr/bin/env python3
"""Device-timed RNEA / forward dynamics with and without external wrenches
(Python API, inputs as (N, n) / (N, n, 6) tensors).  Usage: fext_time.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_04310_b200 as vd  # noqa: E402


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
    for robot, N in (("tree29", 262144), ("chain7", 4194304)):
        m = vd.robots.by_name(robot)
        dm = vd.DeviceModel(m, 0)
        n = m.dof()
        for dt in (torch.float64, torch.float32):
            q, qd, x = [((torch.rand((N, n), device="cuda", dtype=torch.float64) * 2 - 1) * np.pi).to(dt)
                        for _ in range(3)]
            fext = torch.rand((N, n, 6), device="cuda", dtype=torch.float64).to(dt)
            # the C-ABI alone on plane-layout buffers (no host-side transposes)
            lib = vd._lib.load()
            code = 0 if dt == torch.float64 else 1
            P = [t.t().contiguous() for t in (q, qd, x)]
            F = fext.reshape(N, 6 * n).t().contiguous()
            out = torch.empty((n, N), dtype=dt, device="cuda")
            st = torch.empty(N, dtype=torch.int32, device="cuda")
            s = None
            for nm, fx in (("abi rnea", None), ("abi rnea_fext", F)):
                ms = timeit(lambda: lib.vd_rnea(dm.handle, code, N, P[0].data_ptr(), P[1].data_ptr(), P[2].data_ptr(),
                                                N, None, None if fx is None else fx.data_ptr(), out.data_ptr(), N, s))
                print(robot, N, str(dt)[6:], nm, round(ms, 4), "ms", flush=True)
            for nm, fx in (("abi aba", None), ("abi aba_fext", F)):
                ms = timeit(lambda: lib.vd_aba(dm.handle, code, N, P[0].data_ptr(), P[1].data_ptr(), P[2].data_ptr(),
                                               N, None, None if fx is None else fx.data_ptr(), out.data_ptr(), N,
                                               st.data_ptr(), s))
                print(robot, N, str(dt)[6:], nm, round(ms, 4), "ms", flush=True)
            for nm, fn in (("rnea", lambda: vd.rnea(dm, q, qd, x)),
                           ("rnea_fext", lambda: vd.rnea(dm, q, qd, x, fext=fext)),
                           ("aba", lambda: vd.forward_dynamics(dm, q, qd, x, return_status=True)),
                           ("aba_fext", lambda: vd.forward_dynamics(dm, q, qd, x, fext=fext, return_status=True))):
                print(robot, N, str(dt)[6:], nm, round(timeit(fn), 4), "ms", flush=True)


if __name__ == "__main__":
    main()

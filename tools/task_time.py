#!/usr/bin/env python3
"""Device-timed Jacobian / diff-IK / manipulability (and its JVP) through the Python API.

Usage: python tools/task_time.py [N ...]   (chain7 frame `ee`, tree29 `l_palm`)
"""
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
    sizes = [int(a) for a in sys.argv[1:]] or [4096, 32768, 4194304]
    for robot, frame in (("chain7", "ee"), ("tree29", "l_palm")):
        m = vd.robots.by_name(robot)
        dm = vd.DeviceModel(m, 0)
        n = m.dof()
        pose0 = vd.frame_transform(dm, torch.zeros((1, n), dtype=torch.float64, device="cuda"), frame).cpu().numpy()[0]
        R = pose0[:9].reshape(3, 3, order="F")
        tgt = vd.TaskTarget(frame, (R.tolist(), pose0[9:].tolist()))
        for N in sizes:
            if robot == "tree29" and N > 1048576:
                continue
            for dt in (torch.float64, torch.float32):
                q = ((torch.rand((N, n), dtype=torch.float64, device="cuda") * 2 - 1) * np.pi).to(dt)
                calls = {"jacobian": lambda: vd.geometric_jacobian(dm, q, frame),
                         "diff_ik": lambda: vd.diff_ik_step(dm, q, tgt, 0.01),
                         "manipulability": lambda: vd.manipulability(dm, q, frame),
                         "manipulability_jvp": lambda: vd.manipulability_jvp(dm, q, q, frame)}
                for op, fn in calls.items():
                    ms = timeit(fn)
                    print(json.dumps({"robot": robot, "op": op, "dtype": str(dt)[6:], "N": N, "ms": round(ms, 4)}),
                          flush=True)


if __name__ == "__main__":
    main()

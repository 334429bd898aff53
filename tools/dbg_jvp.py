"""Debug helper: run each JVP entry point once and report the first failing one."""
import sys
import numpy as np
import torch
import paper_2604_04310_b200 as vd

name = sys.argv[1] if len(sys.argv) > 1 else "chain7"
for generic in (False, True):
    dm = vd.DeviceModel(vd.robots.by_name(name), 0, generic=generic)
    n = dm.dof()
    q = torch.rand((256, n), dtype=torch.float64, device="cuda")
    for op in ("fk", "rnea", "crba", "aba"):
        try:
            if op == "fk":
                vd.forward_kinematics_jvp(dm, q, q)
            elif op == "rnea":
                vd.rnea_jvp(dm, q, q, q, q, q, q)
            elif op == "crba":
                vd.crba_jvp(dm, q, q)
            else:
                vd.forward_dynamics_jvp(dm, q, q, q, q, q, q, return_status=True)
            torch.cuda.synchronize()
            print(name, generic, op, "ok", flush=True)
        except Exception as e:
            print(name, generic, op, "FAIL", e, flush=True)
            sys.exit(1)

"""Out-of-bounds guards for every device entry point of the C-ABI.

compute-sanitizer is not available on the GPU pool, so bounds are checked
the direct way: every output buffer gets ld_out > N and one extra plane, all
pre-filled with a NaN sentinel; after the call the padding columns, the
extra plane and the status tail must still hold the sentinel, and every
output plane must have been written.  Inputs are read with ld_in > N from buffers
whose padding holds NaN as well, so a read past column N - 1 or of a wrong
plane shows up as a non-finite output; the strided results must equal the
dense (ld = N) call bitwise.  Ragged N (not a multiple of the 128-thread CTA)
exercises the tail lanes of the persistent kernels.
"""
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N = 1001
PAD_IN, PAD_OUT = 19, 33
FRAMES = {"chain7": "ee", "tree29": "l_palm", "humanoid23": "l_palm"}
CASES = [("chain7", False), ("chain7", True), ("tree29", False), ("humanoid23", False)]


def _planes(n, ld, dtype, seed, scale=np.pi):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.full((n, ld), float("nan"), dtype=torch.float64, device="cuda")
    x[:, :N] = (torch.rand((n, N), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) * scale
    return x.to(dtype)


def _ops(vd, lib, name, m, dm, n, dtype):
    """name -> (output plane counts, callable(ins, ld_in, outs, ld_out, status) -> rc)."""
    code = 0 if dtype == torch.float64 else 1
    h = dm.handle
    frame = m.frame_index(FRAMES[name])
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
    T = vd._lib.TaskParams()
    T.frame = frame
    for k in range(9):
        T.target[k] = 1.0 if k in (0, 4, 8) else 0.0
    for k in range(6):
        T.kp[k] = 1.0
    T.damping = 0.05
    g3 = (ctypes.c_double * 3)(0.0, 0.0, 9.81)
    s = None
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    nnz = len(m.crba_pattern()[0])
    ops = {
        "fk": ([12 * n], lambda x, li, y, lo, st: lib.vd_fk(h, code, N, p(x[0]), li, p(y[0]), lo, s)),
        "jacobian": ([12, 6 * n], lambda x, li, y, lo, st: lib.vd_jacobian(h, code, N, p(x[0]), li, frame, p(y[0]),
                                                                            p(y[1]), lo, s)),
        "rnea": ([n], lambda x, li, y, lo, st: lib.vd_rnea(h, code, N, p(x[0]), p(x[1]), p(x[2]), li, g3, None,
                                                           p(y[0]), lo, s)),
        "bias": ([n], lambda x, li, y, lo, st: lib.vd_bias(h, code, N, p(x[0]), p(x[1]), li, g3, None, p(y[0]), lo,
                                                           s)),
        "gravity": ([n], lambda x, li, y, lo, st: lib.vd_gravity(h, code, N, p(x[0]), li, g3, p(y[0]), lo, s)),
        "coriolis": ([n], lambda x, li, y, lo, st: lib.vd_coriolis(h, code, N, p(x[0]), p(x[1]), li, p(y[0]), lo, s)),
        "crba": ([n * n], lambda x, li, y, lo, st: lib.vd_crba(h, code, N, p(x[0]), li, p(y[0]), lo, s)),
        "crba_packed": ([nnz], lambda x, li, y, lo, st: lib.vd_crba_packed(h, code, N, p(x[0]), li, p(y[0]), lo, s)),
        "aba": ([n], lambda x, li, y, lo, st: lib.vd_aba(h, code, N, p(x[0]), p(x[1]), p(x[2]), li, g3, None, p(y[0]),
                                                         lo, st.data_ptr(), s)),
        "dynamics": ([n * n, n, n], lambda x, li, y, lo, st: lib.vd_dynamics(h, code, N, p(x[0]), p(x[1]), p(x[2]),
                                                                              li, g3, p(y[0]), p(y[1]), p(y[2]), lo,
                                                                              st.data_ptr(), s)),
        "osc": ([n, 36], lambda x, li, y, lo, st: lib.vd_osc(h, code, N, p(x[0]), p(x[1]), li, ctypes.byref(P),
                                                             p(y[0]), p(y[1]), lo, st.data_ptr(), s)),
        "diff_ik": ([n, 6], lambda x, li, y, lo, st: lib.vd_diff_ik(h, code, N, p(x[0]), li, ctypes.byref(T),
                                                                    p(y[0]), p(y[1]), lo, st.data_ptr(), s)),
        "fk_jvp": ([12 * n, 12 * n], lambda x, li, y, lo, st: lib.vd_fk_jvp(h, code, N, p(x[0]), p(x[3]), li,
                                                                             p(y[0]), p(y[1]), lo, s)),
        "rnea_jvp": ([n, n], lambda x, li, y, lo, st: lib.vd_rnea_jvp(h, code, N, p(x[0]), p(x[1]), p(x[2]), p(x[3]),
                                                                      p(x[4]), p(x[5]), li, g3, None, p(y[0]),
                                                                      p(y[1]), lo, s)),
        "crba_jvp": ([n * n, n * n], lambda x, li, y, lo, st: lib.vd_crba_jvp(h, code, N, p(x[0]), p(x[3]), li,
                                                                               p(y[0]), p(y[1]), lo, s)),
        "aba_jvp": ([n, n], lambda x, li, y, lo, st: lib.vd_aba_jvp(h, code, N, p(x[0]), p(x[1]), p(x[2]), p(x[3]),
                                                                    p(x[4]), p(x[5]), li, g3, None, p(y[0]), p(y[1]),
                                                                    lo, st.data_ptr(), s)),
    }
    # per-state gravity: plane 3's first three rows are the a_g planes (same ld as the inputs)
    ops["rnea_pg"] = ([n], lambda x, li, y, lo, st: lib.vd_rnea_pg(h, code, N, p(x[0]), p(x[1]), p(x[2]), li, p(x[3]),
                                                                   None, p(y[0]), lo, s))
    ops["gravity_pg"] = ([n], lambda x, li, y, lo, st: lib.vd_gravity_pg(h, code, N, p(x[0]), li, p(x[3]), p(y[0]), lo,
                                                                         s))
    ops["aba_pg"] = ([n], lambda x, li, y, lo, st: lib.vd_aba_pg(h, code, N, p(x[0]), p(x[1]), p(x[2]), li, p(x[3]),
                                                                 None, p(y[0]), lo, st.data_ptr(), s))
    ops["dynamics_pg"] = ([n * n, n, n], lambda x, li, y, lo, st: lib.vd_dynamics_pg(
        h, code, N, p(x[0]), p(x[1]), p(x[2]), li, p(x[3]), p(y[0]), p(y[1]), p(y[2]), lo, st.data_ptr(), s))
    # one plane each, no ld_out (as vd_manipulability)
    ops["manip_jvp"] = ([1, 1], lambda x, li, y, lo, st: lib.vd_manipulability_jvp(h, code, N, p(x[0]), p(x[3]), li,
                                                                                   frame, p(y[0]), p(y[1]), s))
    if m.is_serial_chain():
        ops["fk_scan"] = ([12 * n], lambda x, li, y, lo, st: lib.vd_fk_scan(h, code, N, p(x[0]), li, p(y[0]), lo, s))
    return ops


def _run(fn, planes, ins, ld_in, ld_out, dtype):
    outs = [torch.full((k + 1, ld_out), float("nan"), dtype=dtype, device="cuda") for k in planes]
    st = torch.full((N + 7,), -5, dtype=torch.int32, device="cuda")
    rc = fn(ins, ld_in, outs, ld_out, st)
    torch.cuda.synchronize()
    return rc, outs, st


@pytest.mark.parametrize("name,generic", CASES)
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_every_entry_point_stays_in_bounds(vd, cuda, name, generic, dtype):
    m = vd.robots.by_name(name)
    dm = vd.DeviceModel(m, 0, generic=generic)
    n = m.dof()
    lib = vd._lib.load()
    ins_pad = [_planes(n, N + PAD_IN, dtype, 100 + k, scale=np.pi if k < 3 else 1.0) for k in range(6)]
    ins_dense = [x[:, :N].contiguous() for x in ins_pad]
    for op, (planes, fn) in _ops(vd, lib, name, m, dm, n, dtype).items():
        rc, outs, st = _run(fn, planes, ins_pad, N + PAD_IN, N + PAD_OUT, dtype)
        assert rc == 0, (op, lib.vd_last_error())
        for k, y in zip(planes, outs):
            assert torch.isnan(y[:, N:]).all(), (op, "wrote past column N - 1")
            assert torch.isnan(y[k, :]).all(), (op, "wrote past the last output plane")
            assert not torch.isnan(y[:k, :N]).all(dim=1).any(), (op, "an output plane was not written")
        assert (st[N:] == -5).all(), (op, "status written past N")
        rc2, outs2, st2 = _run(fn, planes, ins_dense, N, N, dtype)
        assert rc2 == 0
        for k, y, y2 in zip(planes, outs, outs2):
            # a read of the NaN input padding turns a finite dense result into NaN here
            a, b = torch.nan_to_num(y[:k, :N], nan=1.25e7), torch.nan_to_num(y2[:k, :N], nan=1.25e7)
            assert torch.equal(a, b), (op, "strided result differs from the dense one")
        assert torch.equal(st[:N], st2[:N]), (op, "status differs")

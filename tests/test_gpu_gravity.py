"""Per-state gravity: vd_rnea_pg / vd_bias_pg / vd_gravity_pg /
vd_aba_pg / vd_dynamics_pg read each state's base acceleration a_g from three
planes.  The reference has one GravitySpec per call (dynamics.hpp:35-50), so
the oracle is run once per distinct gravity vector on the states that carry
it; the GPU results must meet the usual parity bars against it, and on the
generated kernels they must equal the per-call entry point bitwise (the same
routine, a_g loaded instead of passed)."""
import numpy as np
import pytest
import torch

from oracle_ffi import Model as OModel
from oracle_ffi import rel_err

pytestmark = pytest.mark.gpu

N = 1001  # ragged: not a multiple of the 128-thread CTA
TOL = {torch.float64: 1e-10, torch.float32: 1e-4}
# (robot, device-model kind): generated kernels, loop kernels, a JIT module
CASES = [("chain7", "spec"), ("tree29", "spec"), ("chain7", "generic"), ("humanoid23", "generic"),
         ("humanoid23", "jit")]
GRAVITIES = np.array([[0.0, 0.0, 9.81], [0.0, 0.0, 0.0], [1.5, -2.0, 7.0], [-3.0, 0.5, 11.0], [0.2, 9.0, -1.0]])


def _setup(vd, name, kind, dtype, seed):
    om = OModel.builtin(name)
    m = vd.robots.by_name(name)
    dm = vd.DeviceModel(m, 0, generic=kind == "generic", jit=kind == "jit")
    if kind == "jit":
        assert dm.uses_jit()
    q, qd, qdd, tau = om.random_states(N, seed, True, True)
    grp = np.random.default_rng(seed).integers(0, len(GRAVITIES), N)
    # the planes hold the dtype's value of each vector, as the per-call path converts gravity3
    G = GRAVITIES.astype(np.float32).astype(np.float64) if dtype == torch.float32 else GRAVITIES
    return om, dm, (q, qd, qdd, tau), grp, G


def _t(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def _np(t):
    return t.double().cpu().numpy()


def _per_group(grp, G, fn, shape):
    """fn(selection, gravity) for every gravity group, scattered back to batch order."""
    out = np.empty(shape)
    for k in range(len(G)):
        sel = grp == k
        if sel.any():
            out[sel] = fn(sel, tuple(G[k]))
    return out


@pytest.mark.parametrize("name,kind", CASES)
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_rnea_family_per_state_gravity(vd, cuda, oracle, name, kind, dtype):
    om, dm, (q, qd, qdd, _), grp, G = _setup(vd, name, kind, dtype, 41)
    n = om.n
    gp = _t(G[grp], dtype)
    z = np.zeros_like(q)
    tq, tqd, tqdd = _t(q, dtype), _t(qd, dtype), _t(qdd, dtype)
    rng = np.random.default_rng(3)
    fext = rng.uniform(-1, 1, (N, n, 6))
    cases = {
        "rnea": (lambda: vd.rnea(dm, tq, tqd, tqdd, gravity=gp),
                 lambda g: vd.rnea(dm, tq, tqd, tqdd, gravity=vd.GravitySpec(g)),
                 lambda s, g: om.rnea(q[s], qd[s], qdd[s], gravity=g)),
        "rnea+fext": (lambda: vd.rnea(dm, tq, tqd, tqdd, gravity=gp, fext=_t(fext, dtype)),
                      lambda g: vd.rnea(dm, tq, tqd, tqdd, gravity=vd.GravitySpec(g), fext=_t(fext, dtype)),
                      lambda s, g: om.rnea(q[s], qd[s], qdd[s], gravity=g, fext=fext[s])),
        "bias": (lambda: vd.bias_forces(dm, tq, tqd, gravity=gp),
                 lambda g: vd.bias_forces(dm, tq, tqd, gravity=vd.GravitySpec(g)),
                 lambda s, g: om.rnea(q[s], qd[s], z[s], gravity=g)),
        "gravity": (lambda: vd.gravity_vector(dm, tq, gravity=gp),
                    lambda g: vd.gravity_vector(dm, tq, gravity=vd.GravitySpec(g)),
                    lambda s, g: om.rnea(q[s], z[s], z[s], gravity=g)),
    }
    for op, (per_state, per_call, ref_fn) in cases.items():
        got = _np(per_state())
        ref = _per_group(grp, G, ref_fn, (N, n))
        assert rel_err(got, ref, axis=1).max() <= TOL[dtype], (op, float(rel_err(got, ref, axis=1).max()))
        if kind != "generic":
            # generated routine: identical arithmetic to the per-call launch
            same = _per_group(grp, G, lambda s, g: _np(per_call(g))[s], (N, n))
            if (name, kind) == ("chain7", "spec"):
                # the per-call Panda RNEA family runs the double-buffered-input
                # kernel (k_gen_db), per-state gravity the plain one (launch_t):
                # the same routine compiled twice, so ptxas may contract
                # differently; equal to rounding
                tol = 1e-13 if dtype == torch.float64 else 1e-5
                assert rel_err(got, same, axis=1).max() <= tol, op
            else:
                assert np.array_equal(got, same), op


@pytest.mark.parametrize("name,kind", CASES)
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_aba_per_state_gravity(vd, cuda, oracle, name, kind, dtype):
    om, dm, (q, qd, qdd, _), grp, G = _setup(vd, name, kind, dtype, 42)
    n = om.n
    gp = _t(G[grp], dtype)
    # τ = ID(q, q̇, q̈) under each state's own gravity: FD must give q̈ back
    tau = _per_group(grp, G, lambda s, g: om.rnea(q[s], qd[s], qdd[s], gravity=g), (N, n))
    tq, tqd, ttau = _t(q, dtype), _t(qd, dtype), _t(tau, dtype)
    got, status = vd.forward_dynamics(dm, tq, tqd, ttau, gravity=gp, return_status=True)
    assert int(status.abs().max()) == 0
    got = _np(got)
    ref = _per_group(grp, G, lambda s, g: om.forward_dynamics(q[s], qd[s], tau[s], gravity=g)[0], (N, n))
    M = om.crba(q)
    cond = np.linalg.cond(M)
    # DESIGN.md §Parity policy: n·ε·κ(M) bound everywhere, the flat bar on
    # well-conditioned states
    eps = np.finfo(np.float64 if dtype == torch.float64 else np.float32).eps
    bound = np.maximum(TOL[dtype], n * eps * cond)
    well = cond < (1e5 if dtype == torch.float64 else 1e3)
    err = rel_err(got, ref, axis=1)
    assert np.all(err <= bound) and err[well].max(initial=0) <= TOL[dtype]
    if dtype == torch.float64:
        # normwise backward error of M q̈ = τ − bias(g_i) on every state
        bias = _per_group(grp, G, lambda s, g: om.rnea(q[s], qd[s], np.zeros((int(s.sum()), n)), gravity=g), (N, n))
        r = np.einsum("nij,nj->ni", M, got) + bias - tau
        be = np.abs(r).max(1) / (np.abs(M).max((1, 2)) * np.abs(got).max(1) + np.abs(tau - bias).max(1))
        assert be.max() <= 1e-12
    if kind != "generic":
        per_call = lambda s, g: _np(vd.forward_dynamics(dm, tq, tqd, ttau, gravity=vd.GravitySpec(g)))[s]  # noqa: E731
        same = _per_group(grp, G, per_call, (N, n))
        if (name, kind) == ("chain7", "spec"):
            # the per-call Panda ABA is the double-buffered-input kernel, per-state
            # gravity the plain one (launch_t): the same routine compiled twice,
            # so ptxas may contract differently; equal to rounding (× κ(M))
            assert np.all(rel_err(got, same, axis=1) <= bound)
        else:
            assert np.array_equal(got, same)
    # fused entry point: M, bias and q̈ with per-state gravity
    Mg, b, a, st = vd.dynamics(dm, tq, tqd, ttau, gravity=gp)
    assert int(st.abs().max()) == 0
    bias_ref = _per_group(grp, G, lambda s, g: om.rnea(q[s], qd[s], np.zeros((int(s.sum()), n)), gravity=g), (N, n))
    assert rel_err(_np(b), bias_ref, axis=1).max() <= TOL[dtype]
    assert rel_err(_np(Mg).reshape(N, -1), M.reshape(N, -1), axis=1).max() <= TOL[dtype]
    err = rel_err(_np(a), ref, axis=1)
    assert np.all(err <= bound) and err[well].max(initial=0) <= TOL[dtype]


def test_per_state_gravity_argument_errors(vd, cuda):
    m = vd.robots.by_name("chain7")
    dm = vd.DeviceModel(m, 0)
    q = torch.zeros((8, 7), dtype=torch.float64, device="cuda")
    with pytest.raises(vd.DimensionError):
        vd.rnea(dm, q, q, q, gravity=torch.zeros((7, 3), dtype=torch.float64, device="cuda"))
    lib = vd._lib.load()
    import ctypes

    p = ctypes.c_void_p(q.data_ptr())
    rc = lib.vd_rnea_pg(dm.handle, 0, 8, p, p, p, 8, None, None, p, 8, None)
    assert rc != 0 and b"gravity_planes" in lib.vd_last_error()
    # N = 0: nothing to read
    e = torch.zeros((0, 7), dtype=torch.float64, device="cuda")
    assert vd.rnea(dm, e, e, e, gravity=torch.zeros((0, 3), dtype=torch.float64, device="cuda")).shape == (0, 7)

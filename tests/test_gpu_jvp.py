"""GPU parity of the forward-mode JVP kernels (vd_*_jvp)
against the oracle's dual-number evaluation of the reference algorithms
(oracle/orc_dual.hpp, pinned by finite differences in test_oracle_jvp.py).
Values and tangents are both checked: fp64 ≤ 1e-10, fp32 ≤ 1e-4 (vs the fp64
oracle at the fp32-rounded inputs), rel_err of helpers.hpp:67-72.  Forward
dynamics tangents carry M⁻¹ twice (dq̈ = M⁻¹(dτ − dc − dM q̈)), so their bound
scales with κ(M)²; well-conditioned instances meet the flat bar."""
import numpy as np
import pytest
import torch

from oracle_ffi import Model as OModel
from oracle_ffi import rel_err
from urdf_gen import random_urdf

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
TOL32 = 1e-4
ROBOTS = ["chain7", "tree29", "humanoid23"]


def _t(a, dtype=torch.float64):
    return None if a is None else torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def _np(t):
    return t.double().cpu().numpy()


@pytest.fixture(scope="module")
def omodels(oracle):
    return {n: OModel.builtin(n) for n in ROBOTS}


def _case(om, N, seed):
    q, qd, qdd, tau = om.random_states(N, seed, True, True)
    rng = np.random.default_rng(seed)
    return q, qd, qdd, tau, [rng.standard_normal(q.shape) for _ in range(3)]


def _flat(a):
    return np.asarray(a).reshape(a.shape[0], -1)


@pytest.mark.parametrize("name", ROBOTS)
@pytest.mark.parametrize("generic", [False, True])
def test_kinematics_dynamics_jvp_fp64(vd, cuda, omodels, name, generic):
    om = omodels[name]
    dm = vd.DeviceModel(vd.robots.by_name(name), 0, generic=generic)
    q, qd, qdd, tau, (vq, vqd, vqdd) = _case(om, 1031, 11)
    # FK
    val, tan = vd.forward_kinematics_jvp(dm, _t(q), _t(vq))
    rv, rt = om.jvp("fk", (q,), (vq,))
    assert rel_err(_flat(_np(val)), rv, axis=1).max() <= TOL64
    assert rel_err(_flat(_np(tan)), rt, axis=1).max() <= TOL64
    # RNEA along (q, q̇, q̈)
    val, tan = vd.rnea_jvp(dm, _t(q), _t(qd), _t(qdd), _t(vq), _t(vqd), _t(vqdd))
    rv, rt = om.jvp("rnea", (q, qd, qdd), (vq, vqd, vqdd))
    assert rel_err(_np(val), rv, axis=1).max() <= TOL64
    assert rel_err(_np(tan), rt, axis=1).max() <= TOL64
    # CRBA along q
    val, tan = vd.crba_jvp(dm, _t(q), _t(vq))
    rv, rt = om.jvp("crba", (q,), (vq,))
    assert rel_err(_np(val), rv, axis=1).max() <= TOL64
    assert rel_err(_np(tan), rt, axis=1).max() <= TOL64


@pytest.mark.parametrize("name", ROBOTS)
@pytest.mark.parametrize("generic", [False, True])
def test_forward_dynamics_jvp_fp64(vd, cuda, omodels, name, generic):
    om = omodels[name]
    dm = vd.DeviceModel(vd.robots.by_name(name), 0, generic=generic)
    q, qd, _, tau, (vq, vqd, vtau) = _case(om, 1031, 12)
    val, tan, st = vd.forward_dynamics_jvp(dm, _t(q), _t(qd), _t(tau), _t(vq), _t(vqd), _t(vtau),
                                           return_status=True)
    assert int(st.max()) == 0
    rv, rt, rst = om.jvp("fd", (q, qd, tau), (vq, vqd, vtau))
    assert np.all(rst == 0)
    cond = np.linalg.cond(om.crba(q))
    ev = rel_err(_np(val), rv, axis=1)
    et = rel_err(_np(tan), rt, axis=1)
    assert np.all(ev <= np.maximum(TOL64, 1e-15 * cond)), float(ev.max())
    bound = np.maximum(TOL64, 1e-15 * cond * cond)
    w = int(np.argmax(et / bound))
    assert np.all(et <= bound), (float(et[w]), float(cond[w]))
    well = cond < 1e3
    assert et[well].max(initial=0) <= TOL64


@pytest.mark.parametrize("name", ["chain7", "tree29"])
def test_jvp_fp32(vd, cuda, omodels, name):
    om = omodels[name]
    dm = vd.DeviceModel(vd.robots.by_name(name), 0)
    q, qd, qdd, tau, (vq, vqd, vqdd) = _case(om, 1024, 13)
    r32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    q, qd, qdd, vq, vqd, vqdd = map(r32, (q, qd, qdd, vq, vqd, vqdd))
    f = torch.float32
    val, tan = vd.rnea_jvp(dm, _t(q, f), _t(qd, f), _t(qdd, f), _t(vq, f), _t(vqd, f), _t(vqdd, f))
    rv, rt = om.jvp("rnea", (q, qd, qdd), (vq, vqd, vqdd))
    assert rel_err(_np(val), rv, axis=1).max() <= TOL32
    assert rel_err(_np(tan), rt, axis=1).max() <= TOL32
    val, tan = vd.crba_jvp(dm, _t(q, f), _t(vq, f))
    rv, rt = om.jvp("crba", (q,), (vq,))
    assert rel_err(_np(val), rv, axis=1).max() <= TOL32
    assert rel_err(_np(tan), rt, axis=1).max() <= TOL32
    val, tan = vd.forward_kinematics_jvp(dm, _t(q, f), _t(vq, f))
    rv, rt = om.jvp("fk", (q,), (vq,))
    assert rel_err(_flat(_np(tan)), rt, axis=1).max() <= TOL32


def test_jvp_partial_tangents_fext_gravity(vd, cuda, omodels):
    """NULL tangents are zero; f_ext is a constant input; gravity is honoured."""
    om = omodels["tree29"]
    dm = vd.DeviceModel(vd.robots.tree29(), 0)
    N, n = 257, om.n
    q, qd, qdd, tau, (vq, vqd, _) = _case(om, N, 14)
    rng = np.random.default_rng(3)
    fext = rng.uniform(-3, 3, (N, n, 6))
    g = (0.5, -0.2, 9.5)
    val, tan = vd.rnea_jvp(dm, _t(q), _t(qd), _t(qdd), dqd=_t(vqd), gravity=vd.GravitySpec(g), fext=_t(fext))
    rv, rt = om.jvp("rnea", (q, qd, qdd), (None, vqd, None), gravity=g, fext=fext)
    assert rel_err(_np(val), rv, axis=1).max() <= TOL64
    assert rel_err(_np(tan), rt, axis=1).max() <= TOL64
    # the primal output equals the plain kernel bit for bit in value terms
    assert rel_err(_np(val), _np(vd.rnea(dm, _t(q), _t(qd), _t(qdd), vd.GravitySpec(g), _t(fext))),
                   axis=1).max() <= 1e-13
    val, tan = vd.forward_dynamics_jvp(dm, _t(q), _t(qd), _t(tau), dq=_t(vq), gravity=vd.GravitySpec(g),
                                       fext=_t(fext))
    rv, rt, _ = om.jvp("fd", (q, qd, tau), (vq, None, None), gravity=g, fext=fext)
    cond = np.linalg.cond(om.crba(q))
    assert np.all(rel_err(_np(tan), rt, axis=1) <= np.maximum(TOL64, 1e-15 * cond * cond))
    # zero tangent -> zero output tangent
    _, tz = vd.rnea_jvp(dm, _t(q), _t(qd), _t(qdd))
    assert float(tz.abs().max()) == 0.0


def test_jvp_linearity_and_finite_differences(vd, cuda, omodels):
    om = omodels["chain7"]
    dm = vd.DeviceModel(vd.robots.chain7(), 0)
    q, qd, qdd, tau, (v1, v2, v3) = _case(om, 500, 15)
    a, b = 0.7, -1.3
    _, t1 = vd.crba_jvp(dm, _t(q), _t(v1))
    _, t2 = vd.crba_jvp(dm, _t(q), _t(v2))
    _, t12 = vd.crba_jvp(dm, _t(q), _t(a * v1 + b * v2))
    assert rel_err(_np(t12), a * _np(t1) + b * _np(t2), axis=1).max() <= 1e-12
    # central differences of the device's own ABA (step 1e-6, 1e-5)
    h = 1e-6
    _, tan = vd.forward_dynamics_jvp(dm, _t(q), _t(qd), _t(tau), _t(v1), _t(v2), _t(v3))
    fp = _np(vd.forward_dynamics(dm, _t(q + h * v1), _t(qd + h * v2), _t(tau + h * v3)))
    fm = _np(vd.forward_dynamics(dm, _t(q - h * v1), _t(qd - h * v2), _t(tau - h * v3)))
    cond = np.linalg.cond(om.crba(q))
    e = rel_err(_np(tan), (fp - fm) / (2 * h), axis=1)
    assert np.all(e <= np.maximum(1e-5, 1e-9 * cond))


@pytest.mark.parametrize("seed", range(3))
def test_jvp_random_trees(vd, cuda, oracle, seed):
    text = random_urdf(seed, n=12, branchiness=0.5)
    om = OModel.from_urdf(text)
    dm = vd.DeviceModel(vd.urdf.load_model_from_string(text), 0)
    q, qd, qdd, tau, (vq, vqd, vqdd) = _case(om, 300, 400 + seed)
    _, tan = vd.rnea_jvp(dm, _t(q), _t(qd), _t(qdd), _t(vq), _t(vqd), _t(vqdd))
    assert rel_err(_np(tan), om.jvp("rnea", (q, qd, qdd), (vq, vqd, vqdd))[1], axis=1).max() <= TOL64
    _, tan = vd.crba_jvp(dm, _t(q), _t(vq))
    assert rel_err(_np(tan), om.jvp("crba", (q,), (vq,))[1], axis=1).max() <= TOL64


def test_jvp_errors_and_empty(vd, cuda):
    dm = vd.DeviceModel(vd.robots.chain7(), 0)
    e = torch.empty((0, 7), dtype=torch.float64, device="cuda")
    v, t = vd.rnea_jvp(dm, e, e, e)
    assert v.shape == (0, 7) and t.shape == (0, 7)
    lib = vd._lib.load()
    q = torch.zeros((4, 7), dtype=torch.float64, device="cuda")
    # both outputs NULL
    assert lib.vd_crba_jvp(dm.handle, 0, 4, q.data_ptr(), None, 4, None, None, 4, None) == vd._lib.VD_ERR_INVALID_ARGUMENT
    # ld < N
    assert lib.vd_fk_jvp(dm.handle, 0, 4, q.data_ptr(), None, 2, q.data_ptr(), None, 4,
                         None) == vd._lib.VD_ERR_DIMENSION


@pytest.mark.parametrize("name", ["chain7", "tree29"])
def test_dynamics_derivatives_identities(vd, cuda, omodels, name):
    """jacobian_fwd (autodiff.hpp:67-84) of the batched dynamics from n JVP
    passes: ∂q̈/∂τ = M⁻¹; the implicit-function identity ∂q̈/∂(q, q̇) =
    −M⁻¹ ∂τ/∂(q, q̇) at q̈ = FD(q, q̇, τ); ∂τ/∂q̇ against central finite
    differences of the oracle's RNEA."""
    om = omodels[name]
    dm = vd.DeviceModel(vd.robots.by_name(name), 0)
    n = om.n
    q, qd, _, tau = om.random_states(48, 501, True, True)
    M = om.crba(q)
    cond = np.linalg.cond(M)
    keep = cond < 1e6  # identities through M⁻¹ lose ~κ(M)·ε
    T = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
    dq, dqd, dtau = (x.cpu().numpy() for x in vd.forward_dynamics_derivatives(dm, T(q), T(qd), T(tau)))
    assert np.abs(np.einsum("nij,njk->nik", dtau, M) - np.eye(n))[keep].max() <= 1e-8
    qdd = vd.forward_dynamics(dm, T(q), T(qd), T(tau)).cpu().numpy()
    rq, rqd = (x.cpu().numpy() for x in vd.rnea_derivatives(dm, T(q), T(qd), T(qdd)))
    Minv = np.linalg.inv(M)
    scale = np.maximum(1.0, np.abs(dq).max(axis=(1, 2)))
    assert (np.abs(dq + Minv @ rq).max(axis=(1, 2)) / scale)[keep].max() <= 1e-7
    scale = np.maximum(1.0, np.abs(dqd).max(axis=(1, 2)))
    assert (np.abs(dqd + Minv @ rqd).max(axis=(1, 2)) / scale)[keep].max() <= 1e-7
    # finite differences at a bounded q̈ (at the FD q̈ of an ill-conditioned
    # state |τ| reaches 1e6 and the difference quotient's rounding ~ε|τ|/h)
    _, _, qdd_r, _ = om.random_states(48, 502, True, False)
    _, rqd = (x.cpu().numpy() for x in vd.rnea_derivatives(dm, T(q), T(qd), T(qdd_r)))
    h = 1e-6
    for j in range(n):
        e = np.zeros_like(qd)
        e[:, j] = h
        fd = (om.rnea(q, qd + e, qdd_r) - om.rnea(q, qd - e, qdd_r)) / (2 * h)
        assert np.abs(rqd[:, :, j] - fd).max() / max(1.0, np.abs(fd).max()) <= 1e-6


@pytest.mark.parametrize("name", ["chain7", "tree29"])
def test_jacobian_fwd_combinator(vd, cuda, omodels, name):
    """jacobian_fwd (autodiff.hpp:64-84) over the device JVPs: ∂τ/∂q̈ of the
    dual RNEA is the mass matrix (dynamics.hpp:352-365, the reference's own
    CRBA-column = RNEA(e_i) identity), and jvp along v equals J·v."""
    om = omodels[name]
    dm = vd.DeviceModel(vd.robots.by_name(name), 0)
    n = om.n
    q, qd, qdd, _ = om.random_states(512, 61, True, False)
    tq, tqd, tqdd = _t(q), _t(qd), _t(qdd)
    zero = torch.zeros_like(tq)

    def h(x, dx):
        return vd.rnea_jvp(dm, tq, tqd, x, zero, zero, dx)

    J = vd.jacobian_fwd(h, tqdd)
    assert J.shape == (512, n, n)
    assert rel_err(_np(J).reshape(512, -1), om.crba(q).reshape(512, -1), axis=1).max() <= 1e-10
    v = torch.randn(512, n, dtype=torch.float64, device="cuda")
    _, t = vd.jvp(h, tqdd, v)
    assert rel_err(_np(t), _np(torch.einsum("nij,nj->ni", J, v)), axis=1).max() <= 1e-12


def test_aba_jvp_implicit_tree29(vd, cuda, omodels):
    """G1 ABA-JVP runs the implicit-function form (ABA, RNEA-JVP, ABA at zero
    velocity and gravity; vd_inst_gen.cu aba_jvp_implicit): its value output is
    the plain ABA's bit for bit, values-only and tangents-only calls agree with
    the full call, and a padded output layout (ld_out != ld_in) goes through
    the staged copy."""
    om = omodels["tree29"]
    dm = vd.DeviceModel(vd.robots.tree29(), 0)
    q, qd, _, tau, (vq, vqd, vtau) = _case(om, 700, 21)
    val, tan, st = vd.forward_dynamics_jvp(dm, _t(q), _t(qd), _t(tau), _t(vq), _t(vqd), _t(vtau),
                                           return_status=True)
    assert torch.equal(val, vd.forward_dynamics(dm, _t(q), _t(qd), _t(tau)))
    # tangent along dτ alone is M⁻¹ dτ: the same as ABA(q, 0, dτ) at zero gravity
    _, t_tau = vd.forward_dynamics_jvp(dm, _t(q), _t(qd), _t(tau), dtau=_t(vtau))
    ref = vd.forward_dynamics(dm, _t(q), _t(np.zeros_like(qd)), _t(vtau), vd.GravitySpec((0.0, 0.0, 0.0)))
    assert torch.equal(t_tau, ref)
    # raw C-ABI with ld_out > ld_in: values and tangents land in the padded planes
    import ctypes
    from paper_2604_04310_b200 import _lib
    lib = _lib.load()
    N, n = q.shape
    cols = lambda a: torch.as_tensor(np.ascontiguousarray(a.T), device="cuda")  # noqa: E731  (plane layout)
    Q, QD, TAU, DQ, DQD, DTAU = map(cols, (q, qd, tau, vq, vqd, vtau))
    ldo = N + 37
    out = torch.full((n, ldo), 7.0, dtype=torch.float64, device="cuda")
    dout = torch.full((n, ldo), 7.0, dtype=torch.float64, device="cuda")
    g3 = (ctypes.c_double * 3)(0.0, 0.0, 9.81)  # a_g of GravitySpec.standard()
    torch.cuda.synchronize()
    rc = lib.vd_aba_jvp(dm.handle, 0, N, Q.data_ptr(), QD.data_ptr(), TAU.data_ptr(), DQ.data_ptr(), DQD.data_ptr(),
                        DTAU.data_ptr(), N, g3, None, out.data_ptr(), dout.data_ptr(), ldo, None, None)
    torch.cuda.synchronize()
    assert rc == 0, lib.vd_last_error().decode()
    assert torch.equal(out[:, :N].T, val) and torch.equal(dout[:, :N].T, tan)
    assert float(out[:, N:].min()) == 7.0 and float(dout[:, N:].max()) == 7.0
    # singular-free: statuses all zero, tangents finite
    assert int(st.max()) == 0 and bool(torch.isfinite(tan).all())


@pytest.mark.parametrize("name", ["chain7", "tree29"])
def test_aba_jvp_fp32(vd, cuda, omodels, name):
    """fp32 ABA-JVP against the fp64 oracle at the fp32-rounded inputs: ≤ 1e-4
    on well-conditioned chain7 states; tree29 (κ(M) ≥ 3·10⁴ everywhere, §Parity
    policy) within the κ-scaled bound of a backward-stable fp32 solve."""
    om = omodels[name]
    dm = vd.DeviceModel(vd.robots.by_name(name), 0)
    q, qd, _, tau, (vq, vqd, vtau) = _case(om, 1024, 22)
    r32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    q, qd, tau, vq, vqd, vtau = map(r32, (q, qd, tau, vq, vqd, vtau))
    f = torch.float32
    val, tan = vd.forward_dynamics_jvp(dm, _t(q, f), _t(qd, f), _t(tau, f), _t(vq, f), _t(vqd, f), _t(vtau, f))
    rv, rt, _ = om.jvp("fd", (q, qd, tau), (vq, vqd, vtau))
    cond = np.linalg.cond(om.crba(q))
    ev = rel_err(_np(val), rv, axis=1)
    et = rel_err(_np(tan), rt, axis=1)
    eps32 = 6e-8
    assert np.all(ev <= np.maximum(TOL32, 2 * eps32 * cond)), float(ev.max())
    assert np.all(et <= np.maximum(TOL32, 2 * eps32 * cond * np.sqrt(cond))), float(et.max())
    well = cond < 1e3
    assert et[well].max(initial=0) <= TOL32
    print(name, "fp32 aba_jvp rel err: value max %.2e, tangent max %.2e median %.2e"
          % (ev.max(), et.max(), np.median(et)))

"""GPU parity of per-model JIT modules (jit.py): the generated straight-line
routines of a model that is not a compile-time robot, against the CPU oracle
and against the same model on the loop kernels.  Bars as test_gpu_parity.py
(fp64 1e-10, fp32 1e-4 against the fp64 oracle, rel_err of
proj/tests/helpers.hpp:67-72; forward dynamics with the conditioning-aware
bound of DESIGN.md §Parity policy)."""
import numpy as np
import pytest
import torch

from oracle_ffi import Model as OModel
from oracle_ffi import rel_err
from urdf_gen import random_urdf

pytestmark = pytest.mark.gpu

TOL64, TOL32 = 1e-10, 1e-4
CASES = [("random12", lambda: random_urdf(5, n=12)), ("random16", lambda: random_urdf(11, n=16, branchiness=0.6)),
         ("humanoid23", None)]


def _t(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def _np(t):
    return t.double().cpu().numpy()


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def case(request, vd, oracle):
    name, make = request.param
    if make is None:
        m, om = vd.robots.by_name(name), OModel.builtin(name)
    else:
        text = make()
        m, om = vd.urdf.load_model_from_string(text), OModel.from_urdf(text)
    dm = vd.DeviceModel(m, 0, jit=True)
    assert dm.specialization() == 0 and dm.uses_jit()
    generic = vd.DeviceModel(m, 0, generic=True)
    assert not generic.uses_jit()
    return m, om, dm, generic


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_jit_dynamics_match_oracle(vd, cuda, case, dtype):
    m, om, dm, generic = case
    n = om.n
    tol = TOL64 if dtype == torch.float64 else TOL32
    q, qd, qdd, tau = om.random_states(1537, 31, True, True)
    rng = np.random.default_rng(3)
    fext = rng.uniform(-1, 1, (1537, n, 6))
    g = (0.3, -0.2, 9.5)
    G = vd.GravitySpec(g)
    T = lambda a: _t(a, dtype)  # noqa: E731
    assert rel_err(_np(vd.rnea(dm, T(q), T(qd), T(qdd), G)), om.rnea(q, qd, qdd, gravity=g), axis=1).max() <= tol
    assert rel_err(_np(vd.rnea(dm, T(q), T(qd), T(qdd), G, T(fext))), om.rnea(q, qd, qdd, gravity=g, fext=fext),
                   axis=1).max() <= tol
    z = np.zeros_like(q)
    assert rel_err(_np(vd.bias_forces(dm, T(q), T(qd), G)), om.rnea(q, qd, z, gravity=g), axis=1).max() <= tol
    assert rel_err(_np(vd.gravity_vector(dm, T(q), G)), om.rnea(q, z, z, gravity=g), axis=1).max() <= tol
    assert rel_err(_np(vd.coriolis_vector(dm, T(q), T(qd))), om.rnea(q, qd, z, gravity=(0, 0, 0)),
                   axis=1).max() <= tol
    M = om.crba(q)
    assert rel_err(_np(vd.crba(dm, T(q))), M, axis=1).max() <= tol
    rows, cols = m.crba_pattern()
    assert rel_err(_np(vd.crba_packed(dm, T(q))), M[:, rows, cols], axis=1).max() <= tol
    assert rel_err(_np(vd.forward_kinematics(dm, T(q))), om.fk(q), axis=1).max() <= tol
    for fx in (None, fext):
        got = _np(vd.forward_dynamics(dm, T(q), T(qd), T(tau), G, None if fx is None else T(fx)))
        ref, st = om.forward_dynamics(q, qd, tau, gravity=g, fext=fx)
        assert np.all(st == 0)
        err = rel_err(got, ref, axis=1)
        eps = np.finfo(np.float64 if dtype == torch.float64 else np.float32).eps
        cond = np.linalg.cond(M)
        assert np.all(err <= np.maximum(tol, n * eps * cond))
        assert err[cond < 1e5].max(initial=0) <= tol


def test_jit_matches_loop_kernels(vd, cuda, case):
    """Same model, JIT module vs the loop kernels, fp64: the two are separate
    evaluations of the same recursions (agreement to rounding)."""
    m, om, dm, generic = case
    q, qd, qdd, tau = om.random_states(999, 32, True, True)
    a = _np(vd.forward_dynamics(dm, _t(q), _t(qd), _t(tau)))
    b = _np(vd.forward_dynamics(generic, _t(q), _t(qd), _t(tau)))
    cond = np.linalg.cond(om.crba(q))
    assert np.all(rel_err(a, b, axis=1) <= np.maximum(1e-10, om.n * 1e-16 * cond))
    assert rel_err(_np(vd.rnea(dm, _t(q), _t(qd), _t(qdd))), _np(vd.rnea(generic, _t(q), _t(qd), _t(qdd))),
                   axis=1).max() <= 1e-12


def test_jit_host_batch_api(vd, cuda, case):
    """batch_* (batch.hpp:128-165) on host buffers through a model with a JIT
    module attached: the per-device contexts pick the module up."""
    m, om, dm, generic = case
    b = vd.random_states(m, 5000, 77, True, True)
    tau = vd.batch_rnea(m, b)
    assert rel_err(tau, om.rnea(b.q, b.qd, b.qdd), axis=1).max() <= TOL64
    b.tau = tau
    qdd = vd.batch_forward_dynamics(m, b)
    assert rel_err(qdd, b.qdd, axis=1).max() <= 1e-8  # FD∘ID roundtrip (test_dynamics.cpp:335-351)


@pytest.fixture(scope="module")
def task_case(vd, oracle):
    """humanoid23 with a JIT module that also carries its `l_palm` tasks."""
    m, om = vd.robots.by_name("humanoid23"), OModel.builtin("humanoid23")
    dm = vd.DeviceModel(m, 0, jit=True, jit_frames=("l_palm",))
    assert dm.uses_jit()
    return m, om, dm


def test_jit_task_routines_match_oracle(vd, cuda, task_case):
    """OSC (osc_step, control.hpp:108-155), geometric Jacobian
    (kinematics.hpp:108-136), diff-IK (control.hpp:79-97) and manipulability
    (kinematics.hpp:138-153) from the module's generated routines, fp64,
    against the oracle with the conditioning-aware bounds of
    test_gpu_parity.test_osc_fp64 / test_gpu_task."""
    m, om, dm = task_case
    frame, N = "l_palm", 1024
    q, qd, _, _ = om.random_states(N, 93, False, False)
    q0 = np.zeros((1, om.n))
    pose0, _ = om.jacobian(q0, frame)
    R0, p0 = pose0[0, :9].reshape(3, 3, order="F"), pose0[0, 9:]
    tau_ref, lam_ref, st_ref = om.osc(q, qd, frame, R0, p0, [100.0] * 6, [20.0] * 6, [0.0] * 6, np.zeros(om.n),
                                      10.0, 2.0)
    tgt = vd.TaskTarget(frame, (R0, p0), vd.TaskGains.uniform(100.0, 20.0))
    tau, lam, st = vd.osc_step(dm, _t(q), _t(qd), tgt, np.zeros(om.n), vd.PostureGains(10.0, 2.0),
                               return_lambda=True, return_status=True)
    st = st.cpu().numpy()
    assert np.all(st == st_ref)
    ok = st == 0
    kappa = np.linalg.cond(om.crba(q)) * np.linalg.cond(lam_ref)
    bound = np.maximum(TOL64, 1e-16 * kappa)
    assert np.all(rel_err(_np(tau), tau_ref, axis=1)[ok] <= bound[ok])
    assert np.all(rel_err(_np(lam).reshape(N, -1), lam_ref.reshape(N, -1), axis=1)[ok] <= np.maximum(bound[ok], 1e-10))
    pose_ref, J_ref = om.jacobian(q, frame)
    assert rel_err(_np(vd.geometric_jacobian(dm, _t(q), frame)), J_ref, axis=1).max() <= TOL64
    assert rel_err(_np(vd.frame_transform(dm, _t(q), frame)), pose_ref, axis=1).max() <= TOL64
    w = _np(vd.manipulability(dm, _t(q), frame))
    assert rel_err(w[:, None], om.manipulability(q, frame)[:, None], axis=1).max() <= 1e-9
    kp, ff, damping = [5.0, 4.0, 3.0, 2.0, 1.5, 1.0], [0.1, -0.2, 0.3, 0.01, 0.02, -0.03], 1e-2
    qd_ref, err_ref = om.diff_ik(q, frame, R0, p0, kp, ff, damping)
    qd_got, err = vd.diff_ik_step(dm, _t(q), vd.TaskTarget(frame, (R0, p0), vd.TaskGains(kp=kp), twist_ff=ff),
                                  damping, return_error=True)
    G = J_ref @ np.swapaxes(J_ref, 1, 2) + damping * damping * np.eye(6)
    theta = np.linalg.norm(err_ref[:, :3], axis=1)
    klog = np.maximum(1.0, 1.0 / np.maximum(np.pi - theta, 1e-6) ** 2)
    assert np.all(rel_err(_np(qd_got), qd_ref, axis=1) <= np.maximum(TOL64, 1e-16 * np.linalg.cond(G) * klog))
    # manipulability JVP (the module's ManipJvp routine) against the oracle's
    # jvp_scalar, with test_gpu_task.test_manipulability_jvp's κ(J Jᵀ) bound
    w2, dw = (_np(t) for t in vd.manipulability_jvp(dm, _t(q), _t(qd), frame))
    rw, rdw = om.manipulability_jvp(q, qd, frame)
    kappa_j = np.linalg.cond(J_ref @ np.swapaxes(J_ref, 1, 2))
    e = rel_err(dw[:, None], rdw[:, None], axis=1)
    assert rel_err(w2[:, None], rw[:, None], axis=1).max() <= 1e-9
    assert np.all(e <= np.maximum(TOL64, 32 * 2.2e-16 * kappa_j)) and e[kappa_j < 1e3].max() <= TOL64


def _osc_ref_and_got(vd, om, dm, frame, N, seed, dtype):
    q, qd, _, _ = om.random_states(N, seed, False, False)
    pose0, _ = om.jacobian(np.zeros((1, om.n)), frame)
    R0, p0 = pose0[0, :9].reshape(3, 3, order="F"), pose0[0, 9:]
    tau_ref, lam_ref, st_ref = om.osc(q, qd, frame, R0, p0, [100.0] * 6, [20.0] * 6, [0.0] * 6, np.zeros(om.n),
                                      10.0, 2.0)
    tgt = vd.TaskTarget(frame, (R0, p0), vd.TaskGains.uniform(100.0, 20.0))
    tau, lam, st = vd.osc_step(dm, _t(q, dtype), _t(qd, dtype), tgt, np.zeros(om.n), vd.PostureGains(10.0, 2.0),
                               return_lambda=True, return_status=True)
    return q, _np(tau), st.cpu().numpy(), tau_ref, lam_ref, st_ref


def test_jit_task_routines_fp32(vd, cuda, task_case):
    """fp32 OSC from the JIT module against the fp64 oracle: forward error
    bounded by ε₃₂·κ(M)·κ(J M⁻¹ Jᵀ + εI), flat 1e-4 where that is small
    (test_gpu_parity.test_osc_fp32's bound)."""
    m, om, dm = task_case
    q, tau, st, tau_ref, lam_ref, st_ref = _osc_ref_and_got(vd, om, dm, "l_palm", 1024, 95, torch.float32)
    ok = (st == 0) & (st_ref == 0)
    assert ok.mean() > 0.99
    kappa = np.linalg.cond(om.crba(q)) * np.linalg.cond(lam_ref)
    eps = np.finfo(np.float32).eps
    e = rel_err(tau, tau_ref, axis=1)
    assert np.all(e[ok] <= np.maximum(TOL32, om.n * eps * kappa[ok]))
    well = ok & (kappa * eps < 1e-6)
    assert e[well].max(initial=0) <= TOL32


def test_jit_serial_chain_tasks(vd, cuda, oracle):
    """A serial random chain: its JIT module's OSC is the M-based (LTL) form
    (codegen picks it for chains), Jacobian and dynamics against the oracle."""
    text = random_urdf(23, n=9, branchiness=0.0)
    m, om = vd.urdf.load_model_from_string(text), OModel.from_urdf(text)
    assert m.is_serial_chain()
    dm = vd.DeviceModel(m, 0, jit=True, jit_frames=("tool",))
    assert dm.uses_jit()
    q, tau, st, tau_ref, lam_ref, st_ref = _osc_ref_and_got(vd, om, dm, "tool", 1024, 97, torch.float64)
    assert np.all(st == st_ref)
    ok = st == 0
    kappa = np.linalg.cond(om.crba(q)) * np.linalg.cond(lam_ref)
    assert np.all(rel_err(tau, tau_ref, axis=1)[ok] <= np.maximum(TOL64, 1e-16 * kappa[ok]))
    # above the serial-chain scan threshold (32768 states): the module's Jacobian routine
    q, _, _, _ = om.random_states(40000, 98, False, False)
    pose_ref, J_ref = om.jacobian(q, "tool")
    assert rel_err(_np(vd.geometric_jacobian(dm, _t(q), "tool")), J_ref, axis=1).max() <= TOL64
    qd = np.zeros_like(q)
    assert rel_err(_np(vd.rnea(dm, _t(q), _t(qd), _t(q))), om.rnea(q, qd, q), axis=1).max() <= TOL64


def test_builtin_robots_keep_compiled_in_kernels(vd, cuda):
    """jit=True is a no-op for the builtin robots (their generated kernels are
    compiled in), and a forced-generic device model never uses a module."""
    for name, spec in (("chain7", 1), ("tree29", 2)):
        dm = vd.DeviceModel(vd.robots.by_name(name), 0, jit=True)
        assert dm.specialization() == spec and not dm.uses_jit()
    m = vd.urdf.load_model_from_string(random_urdf(5, n=12))
    from paper_2604_04310_b200 import jit

    jit.attach(m)
    assert vd.DeviceModel(m, 0).uses_jit()
    assert not vd.DeviceModel(m, 0, generic=True).uses_jit()

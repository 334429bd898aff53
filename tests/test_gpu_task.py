"""GPU parity of the task-space rows of SURVEY §8(f): diff_ik_step
(control.hpp:79-97) and manipulability (kinematics.hpp:138-153), through the
C-ABI, against the CPU oracle on the same seeded states.  Bars as in
test_gpu_parity.py (fp64 1e-10, fp32 1e-4 with rel_err of helpers.hpp:67-72);
the damped-least-squares solve is bounded by the conditioning of J Jᵀ + λ² I."""
import ctypes

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
FRAMES = {"chain7": "ee", "tree29": "l_palm", "humanoid23": "r_palm"}


def _t(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def _np(t):
    return t.double().cpu().numpy()


@pytest.fixture(scope="module")
def omodels(oracle):
    return {n: OModel.builtin(n) for n in ROBOTS}


def _target(om, frame, seed):
    """A reachable target: the frame pose at another random configuration."""
    q0, _, _, _ = om.random_states(1, seed, False, False)
    pose0, _ = om.jacobian(q0, frame)
    return pose0[0, :9].reshape(3, 3, order="F"), pose0[0, 9:]


def _log_kappa(err):
    """Conditioning of rotation_log (control.hpp:45-68) at the reference error:
    near θ = π the acos form loses accuracy twice — acos' ~ 1/(π − θ) on the
    trace, then sin θ ~ (π − θ) divides — so roundoff in R is amplified by
    ~1/(π − θ)²."""
    theta = np.linalg.norm(err[:, :3], axis=1)
    return np.maximum(1.0, 1.0 / np.maximum(np.pi - theta, 1e-6) ** 2)


def _gram_cond(J, damping):
    G = J @ np.swapaxes(J, 1, 2) + damping * damping * np.eye(6)
    return np.linalg.cond(G)


@pytest.mark.parametrize("name", ROBOTS)
@pytest.mark.parametrize("generic", [False, True])
def test_diff_ik_fp64(vd, cuda, omodels, name, generic):
    om = omodels[name]
    frame = FRAMES[name]
    dm = vd.DeviceModel(vd.robots.by_name(name), 0, generic=generic)
    q, _, _, _ = om.random_states(2048, 91, False, False)
    R, p = _target(om, frame, 92)
    kp = [5.0, 4.0, 3.0, 2.0, 1.5, 1.0]
    ff = [0.1, -0.2, 0.3, 0.01, 0.02, -0.03]
    damping = 1e-2
    qd_ref, err_ref = om.diff_ik(q, frame, R, p, kp, ff, damping)
    tgt = vd.TaskTarget(frame, (R, p), vd.TaskGains(kp=kp), twist_ff=ff)
    qd, err = vd.diff_ik_step(dm, _t(q), tgt, damping, return_error=True)
    klog = _log_kappa(err_ref)
    e_err = rel_err(_np(err), err_ref, axis=1)
    b_err = np.maximum(TOL64, 1e-15 * klog)
    w = int(np.argmax(e_err / b_err))
    assert np.all(e_err <= b_err), (float(e_err[w]), err_ref[w].tolist(), _np(err)[w].tolist())
    _, J = om.jacobian(q, frame)
    bound = np.maximum(TOL64, 1e-16 * _gram_cond(J, damping) * klog)
    e = rel_err(_np(qd), qd_ref, axis=1)
    assert np.all(e <= bound), float((e / bound).max())


@pytest.mark.parametrize("name", ROBOTS)
def test_diff_ik_fp32(vd, cuda, omodels, name):
    om = omodels[name]
    frame = FRAMES[name]
    dm = vd.DeviceModel(vd.robots.by_name(name), 0)
    q, _, _, _ = om.random_states(1024, 93, False, False)
    R, p = _target(om, frame, 94)
    damping = 5e-2
    tgt = vd.TaskTarget(frame, (R, p), vd.TaskGains.uniform(2.0))
    q32 = q.astype(np.float32).astype(np.float64)  # the fp32 kernel sees rounded q
    qd_ref, _ = om.diff_ik(q32, frame, R, p, [2.0] * 6, [0.0] * 6, damping)
    qd = _np(vd.diff_ik_step(dm, _t(q32, torch.float32), tgt, damping))
    _, J = om.jacobian(q32, frame)
    bound = np.maximum(TOL32, 1e-7 * _gram_cond(J, damping) * _log_kappa(om.diff_ik(q32, frame, R, p, [1.0] * 6,
                                                                                 [0.0] * 6, damping)[1]))
    e = rel_err(qd, qd_ref, axis=1)
    assert np.all(e <= bound), float((e / bound).max())


def test_diff_ik_converges(vd, cuda, omodels):
    """Integrating q += dt·q̇ drives the pose error to zero (control.hpp:79-97 used
    as a resolved-rate IK loop), on the device, batch-wide."""
    om = omodels["chain7"]
    dm = vd.DeviceModel(vd.robots.chain7(), 0)
    R, p = _target(om, "ee", 5)
    q0, _, _, _ = om.random_states(1, 5, False, False)
    rng = np.random.default_rng(0)
    q = _t(q0 + 0.05 * rng.standard_normal((256, 7)))
    tgt = vd.TaskTarget("ee", (R, p), vd.TaskGains.uniform(1.0))
    for _ in range(60):
        qd = vd.diff_ik_step(dm, q, tgt, 1e-3)
        q = q + 0.5 * qd
    _, err = vd.diff_ik_step(dm, q, tgt, 1e-3, return_error=True)
    assert float(err.abs().max()) < 1e-8


def test_diff_ik_errors(vd, cuda):
    dm = vd.DeviceModel(vd.robots.chain7(), 0)
    q = torch.zeros((4, 7), dtype=torch.float64, device="cuda")
    tgt = vd.TaskTarget("ee", (np.eye(3), np.zeros(3)))
    with pytest.raises(vd.Error, match="damping must be positive"):
        vd.diff_ik_step(dm, q, tgt, 0.0)
    with pytest.raises(vd.Error, match="nonnegative"):
        vd.diff_ik_step(dm, q, vd.TaskTarget("ee", (np.eye(3), np.zeros(3)), vd.TaskGains.uniform(-1.0)), 1e-2)
    with pytest.raises(vd.UnknownFrameError):
        vd.diff_ik_step(dm, q, vd.TaskTarget("nope", (np.eye(3), np.zeros(3))), 1e-2)
    lib = vd._lib.load()
    P = vd._lib.TaskParams()
    P.frame = 99
    P.damping = 1.0
    assert lib.vd_diff_ik(dm.handle, 0, 4, q.data_ptr(), 4, ctypes.byref(P), q.data_ptr(), None, 4, None,
                          None) == vd._lib.VD_ERR_UNKNOWN_FRAME
    assert lib.vd_manipulability(dm.handle, 0, 4, q.data_ptr(), 4, -1, q.data_ptr(), None) == vd._lib.VD_ERR_UNKNOWN_FRAME
    # N = 0 is a no-op
    assert vd.manipulability(dm, q[:0], "ee").shape == (0,)


@pytest.mark.parametrize("name", ROBOTS)
@pytest.mark.parametrize("generic", [False, True])
def test_manipulability_fp64(vd, cuda, omodels, name, generic):
    om = omodels[name]
    frame = FRAMES[name]
    dm = vd.DeviceModel(vd.robots.by_name(name), 0, generic=generic)
    q, _, _, _ = om.random_states(4096, 95, False, False)
    ref = om.manipulability(q, frame)
    got = _np(vd.manipulability(dm, _t(q), frame))
    assert rel_err(got[:, None], ref[:, None], axis=1).max() <= TOL64
    assert np.all(got >= 0)


def test_manipulability_singular(vd, cuda, omodels):
    """At q = 0 the chain7 arm is stretched out (a kinematic singularity): the
    Gram matrix is singular up to roundoff and both sides agree; a frame on
    the first joint has a rank-1 Jacobian, so w is 0 up to roundoff."""
    om = omodels["chain7"]
    dm = vd.DeviceModel(vd.robots.chain7(), 0)
    q = np.zeros((3, 7))
    got = _np(vd.manipulability(dm, _t(q), "ee"))
    ref = om.manipulability(q, "ee")
    assert np.all(np.abs(got - ref) <= 1e-10)
    m = vd.robots.chain7()
    first = [f[0] for f in m.frames() if f[1] == 0]
    if first:
        assert np.all(np.abs(_np(vd.manipulability(dm, _t(q), first[0]))) <= 1e-12)
        assert np.all(np.abs(om.manipulability(q, first[0])) <= 1e-12)


def test_manipulability_fp32(vd, cuda, omodels):
    om = omodels["tree29"]
    dm = vd.DeviceModel(vd.robots.tree29(), 0)
    q, _, _, _ = om.random_states(2048, 96, False, False)
    q32 = q.astype(np.float32).astype(np.float64)
    ref = om.manipulability(q32, "l_palm")
    got = _np(vd.manipulability(dm, _t(q32, torch.float32), "l_palm"))
    assert rel_err(got[:, None], ref[:, None], axis=1).max() <= TOL32


@pytest.mark.parametrize("seed", range(3))
def test_task_random_trees(vd, cuda, oracle, seed):
    text = random_urdf(seed, n=12, branchiness=0.5)
    om = OModel.from_urdf(text)
    dm = vd.DeviceModel(vd.urdf.load_model_from_string(text), 0)
    q, _, _, _ = om.random_states(500, 200 + seed, False, False)
    assert rel_err(_np(vd.manipulability(dm, _t(q), "tool"))[:, None], om.manipulability(q, "tool")[:, None],
                   axis=1).max() <= TOL64
    R, p = _target(om, "tool", 300 + seed)
    qd_ref, _ = om.diff_ik(q, "tool", R, p, [1.0] * 6, [0.0] * 6, 0.1)
    qd = _np(vd.diff_ik_step(dm, _t(q), vd.TaskTarget("tool", (R, p), vd.TaskGains.uniform(1.0)), 0.1))
    _, J = om.jacobian(q, "tool")
    bound = np.maximum(TOL64, 1e-16 * _gram_cond(J, 0.1) * _log_kappa(om.diff_ik(q, "tool", R, p, [1.0] * 6,
                                                                               [0.0] * 6, 0.1)[1]))
    assert np.all(rel_err(qd, qd_ref, axis=1) <= bound)


# ---------------------------------------------------------------- manipulability JVP / lie_derivative
@pytest.mark.parametrize("name", ROBOTS)
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_manipulability_jvp(vd, cuda, omodels, name, dtype):
    """vd_manipulability_jvp against the oracle's dual-number jvp_scalar of
    manipulability (orc_batch_manip_jvp, pinned by finite differences in
    tests/test_lie.py).  The tangent is compared where w is away from a
    singularity: w is not differentiable where J loses rank, and near it the
    pivot derivatives d√x = dx / 2√x amplify rounding, so the bound is
    32·ε·κ(J Jᵀ) (measured ≤ 0.1·ε·κ on the near-singular states) with the
    flat bar where κ(J Jᵀ) < 1e3."""
    om = omodels[name]
    frame = FRAMES[name]
    dm = vd.DeviceModel(vd.robots.by_name(name), 0)
    q, qd, _, _ = om.random_states(4097, 97, True, False)
    if dtype == torch.float32:
        q, qd = (a.astype(np.float32).astype(np.float64) for a in (q, qd))
    w_ref, dw_ref = om.manipulability_jvp(q, qd, frame)
    w, dw = (_np(t) for t in vd.manipulability_jvp(dm, _t(q, dtype), _t(qd, dtype), frame))
    tol = TOL64 if dtype == torch.float64 else TOL32
    eps = np.finfo(np.float64 if dtype == torch.float64 else np.float32).eps
    _, J = om.jacobian(q, frame)
    kappa = np.linalg.cond(np.einsum("nrk,nck->nrc", J, J))
    well = kappa < 1e3
    assert well.sum() > 1000
    assert np.all(np.isfinite(dw))
    assert rel_err(w[:, None], w_ref[:, None], axis=1).max() <= tol
    err = rel_err(dw[:, None], dw_ref[:, None], axis=1)
    assert np.all(err <= np.maximum(tol, 32 * eps * kappa))
    assert err[well].max() <= tol
    # the value plane is manipulability(); a zero tangent gives a zero derivative
    e_w = rel_err(w[:, None], _np(vd.manipulability(dm, _t(q, dtype), frame))[:, None], axis=1)
    assert np.all(e_w <= np.maximum(tol, 32 * eps * kappa)) and e_w[well].max() <= tol
    lib = vd._lib.load()
    qs = _t(q, dtype).t().contiguous()
    w2, dw2 = torch.empty(4097, dtype=dtype, device="cuda"), torch.full((4097,), 7.0, dtype=dtype, device="cuda")
    assert lib.vd_manipulability_jvp(dm.handle, 0 if dtype == torch.float64 else 1, 4097, qs.data_ptr(), None, 4097,
                                     dm.model.frame_index(frame), w2.data_ptr(), dw2.data_ptr(), None) == 0
    assert torch.count_nonzero(dw2).item() == 0


@pytest.mark.parametrize("name", ["chain7", "tree29"])
def test_lie_derivative_spec_example(vd, cuda, omodels, name):
    """SPEC.md:524 on the GPU: h = manipulability ∘ J(q), f = the forward-
    dynamics drift (q̇, q̈(q, q̇, τ = 0)) on z = (q, q̇): lie_derivative matches
    the central finite-difference directional derivative of the device
    manipulability, rel tol 1e-4."""
    om = omodels[name]
    frame = FRAMES[name]
    dm = vd.DeviceModel(vd.robots.by_name(name), 0)
    n = om.n
    q, qd, _, _ = om.random_states(2048, 98, True, False)
    z = torch.cat([_t(q), _t(qd)], dim=1)
    zero = torch.zeros((2048, n), dtype=torch.float64, device="cuda")

    def drift(z):
        return torch.cat([z[:, n:], vd.forward_dynamics(dm, z[:, :n], z[:, n:], zero)], dim=1)

    def h(z, dz):
        return vd.manipulability_jvp(dm, z[:, :n], dz[:, :n], frame)

    lie = _np(vd.lie_derivative(h, drift, z))
    eps = 1e-6
    fd = (_np(vd.manipulability(dm, _t(q + eps * qd), frame)) - _np(vd.manipulability(dm, _t(q - eps * qd), frame))) / (
        2 * eps)
    w = om.manipulability(q, frame)
    ok = w > 1e-4
    assert ok.sum() > 500
    assert np.all(np.abs(lie - fd)[ok] <= 1e-4 * np.maximum(np.abs(fd[ok]), 1e-3))
    _, ref = om.manipulability_jvp(q, qd, frame)
    assert rel_err(lie[ok, None], ref[ok, None], axis=1).max() <= TOL64

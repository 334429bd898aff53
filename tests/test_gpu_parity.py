"""GPU parity: every kernel, through the C-ABI, against the CPU oracle on the
same seeded inputs.  Bars (BASELINE.json north_star): fp64 rel_err <= 1e-10,
fp32 rel_err <= 1e-4 (vs the fp64 oracle), per instance and per output tensor,
with rel_err as in proj/tests/helpers.hpp:67-72.  Forward dynamics is compared
against the reference's LLT forward dynamics; instances whose mass matrix is
ill-conditioned get a conditioning-scaled bound and a backward-error check
(DESIGN.md §Parity policy)."""
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


def _dm(vd, name, generic=False):
    m = vd.robots.by_name(name)
    return m, vd.DeviceModel(m, 0, generic=generic)


def _t(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def _np(t):
    return t.double().cpu().numpy()


def _states(om, N, seed, with_tau=True):
    return om.random_states(N, seed, True, with_tau)


@pytest.fixture(scope="module")
def omodels(oracle):
    return {n: OModel.builtin(n) for n in ROBOTS}


# ---------------------------------------------------------------- loader / packer on the box
def test_specialization_matches_builtins(vd, cuda):
    for name, spec in (("chain7", 1), ("tree29", 2), ("humanoid23", 0)):
        m, dm = _dm(vd, name)
        assert dm.specialization() == spec
    # a URDF loaded from text with the same content specialises too
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(__file__)), "assets", "chain7.urdf")
    dm = vd.DeviceModel(vd.urdf.load_model(path), 0)
    assert dm.specialization() == 1


# ---------------------------------------------------------------- RNEA family
@pytest.mark.parametrize("name", ROBOTS)
@pytest.mark.parametrize("generic", [False, True])
def test_rnea_fp64(vd, cuda, omodels, name, generic):
    om = omodels[name]
    m, dm = _dm(vd, name, generic)
    q, qd, qdd, _ = _states(om, 4099, 11)
    ref = om.rnea(q, qd, qdd)
    got = _np(vd.rnea(dm, _t(q), _t(qd), _t(qdd)))
    assert rel_err(got, ref, axis=1).max() <= TOL64
    # bias, gravity, coriolis (dynamics.hpp:402-416)
    z = np.zeros_like(q)
    assert rel_err(_np(vd.bias_forces(dm, _t(q), _t(qd))), om.rnea(q, qd, z), axis=1).max() <= TOL64
    assert rel_err(_np(vd.gravity_vector(dm, _t(q))), om.rnea(q, z, z), axis=1).max() <= TOL64
    assert rel_err(_np(vd.coriolis_vector(dm, _t(q), _t(qd))), om.rnea(q, qd, z, gravity=(0, 0, 0)),
                   axis=1).max() <= TOL64


@pytest.mark.parametrize("name", ROBOTS)
def test_rnea_fext_and_gravity(vd, cuda, omodels, name):
    om = omodels[name]
    m, dm = _dm(vd, name)
    N, n = 1000, om.n
    q, qd, qdd, _ = _states(om, N, 12)
    rng = np.random.default_rng(5)
    fext = rng.uniform(-1, 1, (N, n, 6))
    g = (1.5, -2.0, 7.0)
    ref = om.rnea(q, qd, qdd, gravity=g, fext=fext)
    got = _np(vd.rnea(dm, _t(q), _t(qd), _t(qdd), gravity=vd.GravitySpec(g), fext=_t(fext)))
    assert rel_err(got, ref, axis=1).max() <= TOL64


@pytest.mark.parametrize("name", ["chain7", "tree29"])
def test_rnea_fp32(vd, cuda, omodels, name):
    om = omodels[name]
    m, dm = _dm(vd, name)
    q, qd, qdd, _ = _states(om, 4096, 13)
    ref = om.rnea(q, qd, qdd)
    got = _np(vd.rnea(dm, _t(q, torch.float32), _t(qd, torch.float32), _t(qdd, torch.float32)))
    assert rel_err(got, ref, axis=1).max() <= TOL32


# ---------------------------------------------------------------- CRBA
@pytest.mark.parametrize("name", ROBOTS)
@pytest.mark.parametrize("generic", [False, True])
def test_crba_fp64(vd, cuda, omodels, name, generic):
    om = omodels[name]
    m, dm = _dm(vd, name, generic)
    q, _, _, _ = _states(om, 2050, 21, with_tau=False)
    ref = om.crba(q)
    got = _np(vd.crba(dm, _t(q)))
    assert rel_err(got, ref, axis=1).max() <= TOL64
    # exact zeros between branches (test_dynamics.cpp:200-216)
    mask = m.ancestor_mask()
    off = (mask == 0) & (mask.T == 0)
    assert np.all(got[:, off] == 0.0)
    assert np.all(got == np.transpose(got, (0, 2, 1)))


@pytest.mark.parametrize("name", ["chain7", "tree29"])
def test_crba_fp32(vd, cuda, omodels, name):
    om = omodels[name]
    m, dm = _dm(vd, name)
    q, _, _, _ = _states(om, 2048, 22, with_tau=False)
    got = _np(vd.crba(dm, _t(q, torch.float32)))
    assert rel_err(got, om.crba(q), axis=1).max() <= TOL32


@pytest.mark.parametrize("name", ROBOTS)
@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_crba_packed(vd, cuda, omodels, name, generic, dtype):
    """vd_crba_packed: the branch-sparse lower triangle of M (dynamics.hpp:
    331-350) against the oracle, and equal to the dense vd_crba output at the
    packed positions (bitwise for the gather path, to 1e-13 / 1e-5 for the
    separately compiled generated routine)."""
    om = omodels[name]
    m, dm = _dm(vd, name, generic)
    rows, cols = m.crba_pattern()
    mask = m.ancestor_mask()
    assert len(rows) == int(np.tril(mask).sum())
    q, _, _, _ = _states(om, 3001, 23, with_tau=False)  # ragged batch (not a multiple of the CTA)
    qt = _t(q, dtype)
    Mp = vd.crba_packed(dm, qt)
    assert Mp.shape == (3001, len(rows))
    ref = om.crba(q)
    tol = TOL64 if dtype == torch.float64 else TOL32
    assert rel_err(_np(Mp), ref[:, rows, cols], axis=1).max() <= tol
    dense = vd.crba(dm, qt)
    if generic:  # a coalesced gather of the dense M: bitwise
        assert torch.equal(Mp, dense[:, rows, cols])
        assert torch.equal(vd.unpack_crba(m, Mp), dense)
    else:
        # tree29: the packed and dense routines are generated from the same
        # expression graph (gen_crba) but compiled as separate straight-line
        # kernels, so ptxas's FMA contraction may differ in the last bits;
        # chain7 dense M runs the template kernel.  Tight agreement + the
        # identical exact-zero pattern.
        close = 1e-13 if dtype == torch.float64 else 1e-5
        assert rel_err(_np(vd.unpack_crba(m, Mp)), _np(dense), axis=1).max() <= close
        assert torch.equal(vd.unpack_crba(m, Mp) == 0, dense == 0)
    # ld_out > N through the C-ABI (strided planes), and N = 0
    N, nnz = 1000, len(rows)
    out = torch.full((nnz, N + 37), -1.0, dtype=dtype, device="cuda")
    qs = qt[:N].t().contiguous()
    lib = vd._lib.load()
    rc = lib.vd_crba_packed(dm.handle, 0 if dtype == torch.float64 else 1, N, qs.data_ptr(), N, out.data_ptr(), N + 37,
                            None)
    assert rc == 0
    torch.cuda.synchronize()
    assert torch.equal(out[:, :N].t(), Mp[:N])
    assert torch.all(out[:, N:] == -1.0)
    assert lib.vd_crba_packed(dm.handle, 0, 0, qs.data_ptr(), 0, out.data_ptr(), 0, None) == 0


def test_crba_packed_gather_chunks(vd, cuda, omodels):
    """Models without a generated packed routine build dense M in bounded
    pool scratch chunk by chunk (~256 MB of dense planes per chunk) and gather;
    a batch spanning several chunks, written with ld_out > N, equals the dense
    vd_crba output at the packed positions bitwise."""
    m, dm = _dm(vd, "tree29", generic=True)
    rows, cols = m.crba_pattern()
    N, nnz = 90001, len(rows)  # 3 chunks of 39808 states for 29 dof (fp64)
    q = (torch.rand((N, m.dof()), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(7))
         * 2 - 1) * np.pi
    dense = vd.crba(dm, q)
    out = torch.full((nnz, N + 5), -1.0, dtype=torch.float64, device="cuda")
    qs = q.t().contiguous()
    lib = vd._lib.load()
    assert lib.vd_crba_packed(dm.handle, 0, N, qs.data_ptr(), N, out.data_ptr(), N + 5, None) == 0
    torch.cuda.synchronize()
    assert torch.equal(out[:, :N].t(), dense[:, rows, cols])
    assert torch.all(out[:, N:] == -1.0)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_inputs_on_another_device_rejected(vd, cuda):
    m, dm = _dm(vd, "chain7")
    q = torch.zeros((4, 7), dtype=torch.float64, device="cuda:1")
    with pytest.raises(vd.CudaError):
        vd.rnea(dm, q, q, q)


# ---------------------------------------------------------------- forward dynamics (ABA vs LLT oracle)
def _fd_check(om, q, qd, tau, got, tol, name):
    ref, st = om.forward_dynamics(q, qd, tau)
    assert np.all(st == 0)
    err = rel_err(got, ref, axis=1)
    M = om.crba(q)
    cond = np.linalg.cond(M)
    # conditioning-aware bound: forward error of a backward-stable solver
    # scales with κ(M) (DESIGN.md §Parity policy); well-conditioned instances
    # must meet the flat bar.
    eps = np.finfo(np.float64 if tol < 1e-6 else np.float32).eps
    bound = np.maximum(tol, q.shape[1] * eps * cond)  # n·ε·κ(M)
    worst = int(np.argmax(err / bound))
    assert np.all(err <= bound), (name, float(err[worst]), float(cond[worst]), float(bound[worst]))
    well = cond < 1e5
    assert err[well].max(initial=0) <= tol, (name, float(err[well].max(initial=0)))
    # normwise backward error |M q̈ + bias − τ| / (|M| |q̈| + |τ − bias|)
    bias = om.rnea(q, qd, np.zeros_like(q))
    r = np.einsum("nij,nj->ni", M, got) + bias - tau
    be = np.abs(r).max(axis=1) / (np.abs(M).max(axis=(1, 2)) * np.abs(got).max(axis=1) + np.abs(tau - bias).max(axis=1))
    assert be.max() <= (1e-12 if tol < 1e-6 else 1e-4), float(be.max())
    return err, cond


@pytest.mark.parametrize("name", ROBOTS)
@pytest.mark.parametrize("generic", [False, True])
def test_aba_fp64(vd, cuda, omodels, name, generic):
    om = omodels[name]
    m, dm = _dm(vd, name, generic)
    q, qd, _, tau = _states(om, 4099, 31)
    got, status = vd.forward_dynamics(dm, _t(q), _t(qd), _t(tau), return_status=True)
    assert int(status.max()) == 0
    _fd_check(om, q, qd, tau, _np(got), TOL64, name)


@pytest.mark.parametrize("name", ["chain7", "tree29"])
def test_aba_fp32(vd, cuda, omodels, name):
    om = omodels[name]
    m, dm = _dm(vd, name)
    q, qd, _, tau = _states(om, 4096, 32)
    got, status = vd.forward_dynamics(dm, _t(q, torch.float32), _t(qd, torch.float32), _t(tau, torch.float32),
                                      return_status=True)
    _fd_check(om, q, qd, tau, _np(got), TOL32, name)


@pytest.mark.parametrize("name", ROBOTS)
def test_aba_fext(vd, cuda, omodels, name):
    om = omodels[name]
    m, dm = _dm(vd, name)
    N, n = 512, om.n
    q, qd, qdd, _ = _states(om, N, 33)
    rng = np.random.default_rng(7)
    fext = rng.uniform(-5, 5, (N, n, 6))
    g = (0.3, -0.4, 9.0)
    tau = om.rnea(q, qd, qdd, gravity=g, fext=fext)
    ref, st = om.forward_dynamics(q, qd, tau, gravity=g, fext=fext)
    got = _np(vd.forward_dynamics(dm, _t(q), _t(qd), _t(tau), gravity=vd.GravitySpec(g), fext=_t(fext)))
    # FD∘ID roundtrip (test_dynamics.cpp:335-351) and agreement with the oracle
    assert rel_err(got, qdd, axis=1).max() <= 1e-8 or name == "tree29"
    M = om.crba(q)
    well = np.linalg.cond(M) < 1e5
    assert rel_err(got, ref, axis=1)[well].max() <= TOL64


def test_dynamics_fused(vd, cuda, omodels):
    om = omodels["chain7"]
    for dtype, tol in ((torch.float64, TOL64), (torch.float32, TOL32)):
        m, dm = _dm(vd, "chain7")
        q, qd, _, tau = _states(om, 65536 // 16, 41)
        M, b, a, st = vd.dynamics(dm, _t(q, dtype), _t(qd, dtype), _t(tau, dtype))
        assert int(st.max()) == 0
        assert rel_err(_np(M), om.crba(q), axis=1).max() <= tol
        assert rel_err(_np(b), om.rnea(q, qd, np.zeros_like(q)), axis=1).max() <= tol
        ref, _ = om.forward_dynamics(q, qd, tau)
        assert rel_err(_np(a), ref, axis=1).max() <= tol


def test_singular_model_reports_status(vd, cuda):
    # test_dynamics.cpp:372-382: a zero-inertia dof -> SingularInertiaError
    text = """<robot name="g"><link name="base"/>
      <link name="ghost"><inertial><mass value="0"/><inertia ixx="0" ixy="0" ixz="0" iyy="0" iyz="0" izz="0"/>
      </inertial></link>
      <joint name="j" type="revolute"><parent link="base"/><child link="ghost"/><axis xyz="0 0 1"/></joint></robot>"""
    m = vd.urdf.load_model_from_string(text)
    dm = vd.DeviceModel(m, 0)
    z = torch.zeros((3, 1), dtype=torch.float64, device="cuda")
    with pytest.raises(vd.SingularInertiaError):
        vd.forward_dynamics(dm, z, z, z)
    _, st = vd.forward_dynamics(dm, z, z, z, return_status=True)
    assert st.tolist() == [7, 7, 7]


def test_prismatic_free_fall(vd, cuda):
    # test_dynamics.cpp:97-108
    text = """<robot name="p"><link name="base"/>
      <link name="slider"><inertial><mass value="2.5"/><inertia ixx="0" ixy="0" ixz="0" iyy="0" iyz="0" izz="0"/>
      </inertial></link>
      <joint name="lift" type="prismatic"><parent link="base"/><child link="slider"/><axis xyz="0 0 1"/></joint>
      </robot>"""
    dm = vd.DeviceModel(vd.urdf.load_model_from_string(text), 0)
    z = torch.zeros((1, 1), dtype=torch.float64, device="cuda")
    assert abs(float(vd.gravity_vector(dm, z)[0, 0]) - 2.5 * 9.81) < 1e-14 * 2.5 * 9.81
    assert abs(float(vd.forward_dynamics(dm, z, z, z)[0, 0]) + 9.81) < 1e-12


# ---------------------------------------------------------------- kinematics
@pytest.mark.parametrize("name,frame", [("chain7", "ee"), ("tree29", "l_palm"), ("tree29", "head"),
                                         ("humanoid23", "r_palm")])
@pytest.mark.parametrize("generic", [False, True])
def test_fk_and_jacobian(vd, cuda, omodels, name, frame, generic):
    om = omodels[name]
    m, dm = _dm(vd, name, generic)
    q, _, _, _ = _states(om, 4096, 51, with_tau=False)
    fk_ref = om.fk(q)
    fk = _np(vd.forward_kinematics(dm, _t(q)))
    assert rel_err(fk, fk_ref, axis=1).max() <= TOL64
    pose_ref, J_ref = om.jacobian(q, frame)
    pose = _np(vd.frame_transform(dm, _t(q), frame))
    J = _np(vd.geometric_jacobian(dm, _t(q), frame))
    assert rel_err(pose, pose_ref, axis=1).max() <= TOL64
    assert rel_err(J, J_ref, axis=1).max() <= TOL64
    # non-ancestor columns are exactly zero (test_kinematics.cpp:192-209)
    fj = [f for f in m.frames() if f[0] == frame][0][1]
    mask = m.ancestor_mask()
    for j in range(m.dof()):
        if mask[fj, j] == 0:
            assert np.all(J[:, :, j] == 0.0)
    # fp32
    fk32 = _np(vd.forward_kinematics(dm, _t(q, torch.float32)))
    assert rel_err(fk32, fk_ref, axis=1).max() <= TOL32


def test_fk_scan(vd, cuda, omodels, oracle):
    """forward_kinematics_scan (kinematics.hpp:61-86) ≡ sequential FK; rejects trees."""
    om = omodels["chain7"]
    m, dm = _dm(vd, "chain7")
    for N in (1, 5, 4096, 4099):
        q, _, _, _ = _states(om, N, 81 + N, with_tau=False)
        ref = om.fk(q, scan=True)
        assert rel_err(_np(vd.forward_kinematics_scan(dm, _t(q))), ref, axis=1).max() <= 1e-12
        assert rel_err(_np(vd.forward_kinematics_scan(dm, _t(q, torch.float32))), ref, axis=1).max() <= TOL32
    # random serial chains n = 1..16 (test_kinematics.cpp:105-120)
    for n in (1, 3, 8, 9, 16):
        text = random_urdf(500 + n, n=n, branchiness=0.0, fixed_prob=0.0)
        o = OModel.from_urdf(text)
        dmr = vd.DeviceModel(vd.urdf.load_model_from_string(text), 0)
        q, _, _, _ = o.random_states(300, 7, True, False)
        assert rel_err(_np(vd.forward_kinematics_scan(dmr, _t(q))), o.fk(q), axis=1).max() <= 1e-12
    with pytest.raises(vd.UnsupportedStructureError):
        _, dt = _dm(vd, "tree29")
        vd.forward_kinematics_scan(dt, _t(np.zeros((4, 29))))


# ---------------------------------------------------------------- OSC
def _osc_case(vd, om, m, dm, name, N, seed, dtype=torch.float64, frame=None):
    if frame is None:
        frame = "ee" if name == "chain7" else ("l_palm" if name != "humanoid23" else "r_palm")
    q, qd, _, _ = _states(om, N, seed, with_tau=False)
    q0 = np.zeros((1, om.n))
    pose0, _ = om.jacobian(q0, frame)
    R0 = pose0[0, :9].reshape(3, 3, order="F")
    p0 = pose0[0, 9:]
    kp, kd = [100.0] * 6, [20.0] * 6
    posture = np.zeros(om.n)
    tau_ref, lam_ref, st_ref = om.osc(q, qd, frame, R0, p0, kp, kd, [0.0] * 6, posture, 10.0, 2.0)
    tgt = vd.TaskTarget(frame, (R0, p0), vd.TaskGains.uniform(100.0, 20.0))
    tau, lam, st = vd.osc_step(dm, _t(q, dtype), _t(qd, dtype), tgt, posture, vd.PostureGains(10.0, 2.0),
                               return_lambda=True, return_status=True)
    return q, _np(tau), _np(lam), st.cpu().numpy(), tau_ref, lam_ref, st_ref


@pytest.mark.parametrize("name", ROBOTS)
@pytest.mark.parametrize("generic", [False, True])
def test_osc_fp64(vd, cuda, omodels, name, generic):
    om = omodels[name]
    m, dm = _dm(vd, name, generic)
    q, tau, lam, st, tau_ref, lam_ref, st_ref = _osc_case(vd, om, m, dm, name, 1024, 61)
    assert np.all(st == st_ref)
    ok = st == 0
    M = om.crba(q)
    cond = np.linalg.cond(M)
    e_tau = rel_err(tau, tau_ref, axis=1)
    e_lam = rel_err(lam, lam_ref, axis=1)
    # OSC chains two solves: with M (κ(M)) and with J M⁻¹ Jᵀ + εI (κ(Λ⁻¹),
    # large near kinematic singularities of the task frame); the forward error
    # of a backward-stable evaluation scales with their product.
    cond_task = np.linalg.cond(lam_ref)
    kappa = cond * cond_task
    bound = np.maximum(TOL64, 1e-16 * kappa)
    worst = int(np.argmax(e_tau / bound))
    assert np.all(e_tau[ok] <= bound[ok]), (float(e_tau[worst]), float(cond[worst]), float(cond_task[worst]))
    assert np.all(e_lam[ok] <= np.maximum(bound[ok], 1e-10)), float(e_lam.max())
    well = ok & (kappa < 1e6)
    assert e_tau[well].max(initial=0) <= TOL64


# ---------------------------------------------------------------- random trees (generic kernels)
@pytest.mark.parametrize("seed", range(6))
def test_random_urdf_trees(vd, cuda, oracle, seed):
    text = random_urdf(seed, n=12, branchiness=0.5)
    om = OModel.from_urdf(text)
    m = vd.urdf.load_model_from_string(text)
    dm = vd.DeviceModel(m, 0)
    assert dm.specialization() == 0
    n = om.n
    q, qd, qdd, tau = om.random_states(777, 100 + seed, True, True)
    rng = np.random.default_rng(seed)
    fext = rng.uniform(-1, 1, (777, n, 6))
    g = tuple(rng.uniform(-5, 5, 3))
    assert rel_err(_np(vd.rnea(dm, _t(q), _t(qd), _t(qdd), vd.GravitySpec(g), _t(fext))),
                   om.rnea(q, qd, qdd, gravity=g, fext=fext), axis=1).max() <= TOL64
    assert rel_err(_np(vd.crba(dm, _t(q))), om.crba(q), axis=1).max() <= TOL64
    tau2 = om.rnea(q, qd, qdd, gravity=g, fext=fext)
    got = _np(vd.forward_dynamics(dm, _t(q), _t(qd), _t(tau2), vd.GravitySpec(g), _t(fext)))
    assert rel_err(got, qdd, axis=1).max() <= 1e-8  # FD∘ID roundtrip
    assert rel_err(_np(vd.forward_kinematics(dm, _t(q))), om.fk(q), axis=1).max() <= TOL64
    pose_ref, J_ref = om.jacobian(q, "tool")
    assert rel_err(_np(vd.geometric_jacobian(dm, _t(q), "tool")), J_ref, axis=1).max() <= TOL64


# ---------------------------------------------------------------- edge cases
def test_edge_cases(vd, cuda, omodels):
    lib = vd._lib.load()
    m, dm = _dm(vd, "chain7")
    # N = 0 is a no-op
    e = torch.empty((0, 7), dtype=torch.float64, device="cuda")
    assert vd.rnea(dm, e, e, e).shape == (0, 7)
    # N = 1 and ragged N
    om = omodels["chain7"]
    for N in (1, 127, 129, 1000):
        q, qd, qdd, _ = _states(om, N, 70 + N)
        assert rel_err(_np(vd.rnea(dm, _t(q), _t(qd), _t(qdd))), om.rnea(q, qd, qdd), axis=1).max() <= TOL64
    # ld > N through the raw C-ABI: a padded (n, ld) buffer
    N, ld = 100, 160
    q, qd, qdd, _ = _states(om, N, 77)
    pad = lambda a: torch.nn.functional.pad(_t(a).t().contiguous(), (0, ld - N))  # noqa: E731
    Q, QD, QDD = pad(q), pad(qd), pad(qdd)
    out = torch.full((7, ld), 123.0, dtype=torch.float64, device="cuda")
    rc = lib.vd_rnea(dm.handle, 0, N, Q.data_ptr(), QD.data_ptr(), QDD.data_ptr(), ld, None, None, out.data_ptr(), ld,
                     None)
    torch.cuda.synchronize()
    assert rc == 0
    assert rel_err(_np(out[:, :N].t()), om.rnea(q, qd, qdd), axis=1).max() <= TOL64
    assert torch.all(out[:, N:] == 123.0)
    # argument errors map to the reference exception types
    assert lib.vd_rnea(dm.handle, 0, N, Q.data_ptr(), QD.data_ptr(), QDD.data_ptr(), N - 1, None, None,
                       out.data_ptr(), ld, None) == vd._lib.VD_ERR_DIMENSION
    assert lib.vd_rnea(dm.handle, 5, N, Q.data_ptr(), QD.data_ptr(), QDD.data_ptr(), ld, None, None,
                       out.data_ptr(), ld, None) == vd._lib.VD_ERR_INVALID_ARGUMENT
    with pytest.raises(vd.DimensionError):
        vd.rnea(dm, _t(np.zeros((3, 6))), _t(np.zeros((3, 6))), _t(np.zeros((3, 6))))
    with pytest.raises(vd.UnknownFrameError):
        vd.geometric_jacobian(dm, _t(q), "nope")
    # 0-dof model yields empty results (test_dynamics.cpp:415-424)
    m0 = vd.urdf.load_model_from_string(
        '<robot name="z"><link name="base"/><link name="tool"/>'
        '<joint name="mount" type="fixed"><parent link="base"/><child link="tool"/></joint></robot>')
    dm0 = vd.DeviceModel(m0, 0)
    e0 = torch.empty((4, 0), dtype=torch.float64, device="cuda")
    assert vd.rnea(dm0, e0, e0, e0).shape == (4, 0)


# ---------------------------------------------------------------- full-size properties
def test_full_size_properties(vd, cuda):
    """BASELINE configs at full size: FD∘ID roundtrip (test_dynamics.cpp:335-351)
    and CRBA column = RNEA(e_i) (test_dynamics.cpp:153-166) on the device."""
    for name, N in (("chain7", 65536), ("tree29", 262144)):
        m, dm = _dm(vd, name)
        g = torch.Generator(device="cuda").manual_seed(9)
        n = m.dof()
        q = (torch.rand((N, n), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) * np.pi
        qd = (torch.rand((N, n), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) * np.pi
        qdd = (torch.rand((N, n), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) * np.pi
        tau = vd.rnea(dm, q, qd, qdd)
        back, st = vd.forward_dynamics(dm, q, qd, tau, return_status=True)
        err = (back - qdd).abs().amax(dim=1) / torch.clamp(torch.maximum(back.abs().amax(1), qdd.abs().amax(1)), min=1)
        cosb = torch.cos(q[:, 4]).abs() if name == "tree29" else torch.ones(N, device="cuda", dtype=torch.float64)
        assert float(err[cosb > 0.05].max()) <= 1e-8
        M = vd.crba(dm, q[:4096])
        z = torch.zeros_like(q[:4096])
        for i in range(0, n, 3):
            e = torch.zeros_like(z)
            e[:, i] = 1
            col = vd.rnea(dm, q[:4096], z, e, gravity=vd.GravitySpec.zero())
            d = (M[:, :, i] - col).abs().amax(1) / torch.clamp(col.abs().amax(1), min=1)
            assert float(d.max()) <= 1e-9


def test_host_batch_api(vd, cuda, omodels):
    """batch_rnea / batch_crba / batch_forward_dynamics (batch.hpp:128-165) on host buffers."""
    m = vd.robots.tree29()
    b = vd.random_states(m, 3001, 2604, True, True)
    om = omodels["tree29"]
    q, qd, qdd, tau = om.random_states(3001, 2604, True, True)
    assert np.array_equal(b.q, q) and np.array_equal(b.tau, tau)  # bit-identical RNG stream
    assert rel_err(vd.batch_rnea(m, b), om.rnea(q, qd, qdd), axis=1).max() <= TOL64
    Mh = vd.batch_crba(m, b)
    assert rel_err(Mh.reshape(3001, 29, 29, order="C").transpose(0, 2, 1), om.crba(q), axis=1).max() <= TOL64
    b2 = vd.StateBatch(b.q, b.qd, None, om.rnea(q, qd, qdd))
    got = vd.batch_forward_dynamics(m, b2)
    cosb = np.abs(np.cos(q[:, 4]))
    assert rel_err(got, qdd, axis=1)[cosb > 0.05].max() <= 1e-8


def test_host_batch_chunk_plan(vd, cuda, omodels):
    """The host pipeline streams full chunks, then halving chunks over the last
    two chunks' worth (vd_abi.cpp run_shard): with the chunk knob at its
    65 536-state floor, 300 000 Panda states run as 3 full, 4 tapered and one
    remainder chunk, bitwise equal to one device call (pageable numpy buffers
    through the staging path, and pinned torch buffers direct)."""
    import ctypes
    lib = vd._lib.load()
    lib.vdi_set_host_chunk_bytes.argtypes = [ctypes.c_int64]
    lib.vdi_set_host_chunk_bytes.restype = None
    om = omodels["chain7"]
    m, dm = _dm(vd, "chain7")
    N = 300000
    b = vd.random_states(m, N, 77, False, True)
    dev = vd.forward_dynamics(dm, _t(b.q), _t(b.qd), _t(b.tau)).cpu().numpy()
    lib.vdi_set_host_chunk_bytes(1)
    try:
        got = vd.batch_forward_dynamics(m, b)
        assert np.array_equal(got, dev)
        hq, hqd, htau = (torch.as_tensor(np.ascontiguousarray(a.T)).pin_memory() for a in (b.q, b.qd, b.tau))
        hout = torch.empty_like(hq).pin_memory()
        hst = torch.full((N,), -1, dtype=torch.int32).pin_memory()
        devs = (ctypes.c_int * 1)(0)
        rc = lib.vd_batch_forward_dynamics_host(m.handle, N, hq.data_ptr(), hqd.data_ptr(), htau.data_ptr(), None,
                                                hout.data_ptr(), hst.data_ptr(), devs, 1)
        assert rc == 0, lib.vd_last_error().decode()
        assert np.array_equal(hout.numpy().T, dev) and int(hst.abs().max()) == 0
    finally:
        lib.vdi_set_host_chunk_bytes(0)
    idx = np.arange(0, N, 997)
    ref, _ = om.forward_dynamics(b.q[idx], b.qd[idx], b.tau[idx])
    assert rel_err(dev[idx], ref, axis=1).max() <= TOL64


def test_batch_eval(vd, cuda, omodels):
    """batch_eval (batch.hpp:76-126): fn runs once per contiguous shard on its
    device; the concatenation is bitwise identical for any partition (here 1
    and 3 shards on the one GPU) and equals the oracle; N = 0 gives 0 x 0."""
    m = vd.robots.tree29()
    b = vd.random_states(m, 3001, 2605, True, True)
    om = omodels["tree29"]

    def fn(dm, s):
        return torch.cat([vd.rnea(dm, s.q, s.qd, s.qdd), vd.forward_dynamics(dm, s.q, s.qd, s.tau)], dim=1)

    one = vd.batch_eval(m, b, fn)
    three = vd.batch_eval(m, b, fn, devices=[0, 0, 0])
    assert one.shape == (3001, 58) and np.array_equal(one, three)
    assert rel_err(one[:, :29], om.rnea(b.q, b.qd, b.qdd), axis=1).max() <= TOL64
    assert np.array_equal(one[:, :29], vd.batch_rnea(m, b))
    empty = vd.StateBatch(np.zeros((0, 29), order="F"), np.zeros((0, 29), order="F"))
    assert vd.batch_eval(m, empty, fn).shape == (0, 0)
    with pytest.raises(vd.DimensionError):
        vd.batch_eval(m, b, lambda dm, s: s.q[:5])


def test_results_independent_of_batch_position(vd, cuda, omodels):
    """Every instance is computed by the same instruction stream whatever N,
    ld or pointer alignment (TMA tiles, tail tile, plain-staged tiles): shards
    of a batch concatenate bit-identically (batch.hpp:77-81 determinism)."""
    om = omodels["chain7"]
    m, dm = _dm(vd, "chain7")
    N = 4099
    q, qd, _, tau = _states(om, N, 91)
    full = vd.forward_dynamics(dm, _t(q), _t(qd), _t(tau))
    pieces = []
    for lo, hi in ((0, 1), (1, 2050), (2050, 2051), (2051, 4099)):
        pieces.append(vd.forward_dynamics(dm, _t(q[lo:hi]), _t(qd[lo:hi]), _t(tau[lo:hi])))
    assert torch.equal(torch.cat(pieces), full)
    # misaligned planes (odd ld through the raw C-ABI) use the plain-staged path
    lib = vd._lib.load()
    ld = N + 1
    pad = lambda a: torch.nn.functional.pad(_t(a).t().contiguous(), (0, 1))  # noqa: E731
    Q, QD, TA = pad(q), pad(qd), pad(tau)
    out = torch.zeros((7, ld), dtype=torch.float64, device="cuda")
    rc = lib.vd_aba(dm.handle, 0, N, Q.data_ptr(), QD.data_ptr(), TA.data_ptr(), ld, None, None, out.data_ptr(), ld,
                    None, None)
    torch.cuda.synchronize()
    assert rc == 0
    assert torch.equal(out[:, :N].t(), full)
    # same for RNEA
    full_r = vd.rnea(dm, _t(q), _t(qd), _t(tau))
    part_r = torch.cat([vd.rnea(dm, _t(q[a:b]), _t(qd[a:b]), _t(tau[a:b])) for a, b in ((0, 77), (77, 4099))])
    assert torch.equal(part_r, full_r)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_tree29_generated_aba_shards_and_ld(vd, cuda, omodels, dtype):
    """G1 ABA runs the generated straight-line kernel (persistent grid, state
    slots in registers / shared memory / L2 scratch): per-instance results do
    not depend on N, the shard boundaries, the grid size or an odd leading
    dimension, and agree with the loop kernel (generic view)."""
    om = omodels["tree29"]
    m, dm = _dm(vd, "tree29")
    assert dm.specialization() == 2
    N = 70001  # > one persistent wave at 148 SMs x 2..4 CTAs x 128 threads
    q, qd, _, tau = _states(om, N, 95)
    full = vd.forward_dynamics(dm, _t(q, dtype), _t(qd, dtype), _t(tau, dtype))
    pieces = [vd.forward_dynamics(dm, _t(q[a:b], dtype), _t(qd[a:b], dtype), _t(tau[a:b], dtype))
              for a, b in ((0, 1), (1, 33), (33, 40000), (40000, N))]
    assert torch.equal(torch.cat(pieces), full)
    lib = vd._lib.load()
    ld = N + 3
    pad = lambda a: torch.nn.functional.pad(_t(a, dtype).t().contiguous(), (0, 3))  # noqa: E731
    Q, QD, TA = pad(q), pad(qd), pad(tau)
    out = torch.zeros((29, ld), dtype=dtype, device="cuda")
    st = torch.full((N,), -1, dtype=torch.int32, device="cuda")
    rc = lib.vd_aba(dm.handle, 0 if dtype == torch.float64 else 1, N, Q.data_ptr(), QD.data_ptr(), TA.data_ptr(), ld,
                    None, None, out.data_ptr(), ld, st.data_ptr(), None)
    torch.cuda.synchronize()
    assert rc == 0 and int(st.max()) == 0 and int(st.min()) == 0
    assert torch.equal(out[:, :N].t(), full)
    _, dg = _dm(vd, "tree29", True)
    loop = vd.forward_dynamics(dg, _t(q[:4096], dtype), _t(qd[:4096], dtype), _t(tau[:4096], dtype))
    cond = np.linalg.cond(om.crba(q[:4096]))
    d = rel_err(_np(full[:4096]), _np(loop), axis=1)
    eps = float(torch.finfo(dtype).eps)
    assert np.all(d <= np.maximum(1e-10 if dtype == torch.float64 else 1e-4, 29 * eps * cond))


@pytest.mark.parametrize("frame", ["head", "r_foot", "r_palm", "l_hand"])
def test_osc_tree29_frames(vd, cuda, omodels, frame):
    """G1 OSC on other task frames: generated variants (leaf joints and fused
    frames: head on the torso, r_foot, r_palm) and the loop kernel fallback
    (l_hand's joint 23 also carries l_palm, so it is generated too) against
    the oracle's osc_step (control.hpp:108-155)."""
    om = omodels["tree29"]
    m, dm = _dm(vd, "tree29")
    q, tau, lam, st, tau_ref, lam_ref, st_ref = _osc_case(vd, om, m, dm, "tree29", 1024, 63, frame=frame)
    assert np.all(st == st_ref)
    ok = st == 0
    kappa = np.linalg.cond(om.crba(q)) * np.linalg.cond(lam_ref)
    bound = np.maximum(TOL64, 1e-16 * kappa)
    assert np.all(rel_err(tau, tau_ref, axis=1)[ok] <= bound[ok])
    assert np.all(rel_err(lam, lam_ref, axis=1)[ok] <= np.maximum(bound[ok], 1e-10))


@pytest.mark.parametrize("wrap", [0.0, 1e3, 1e7])
def test_aba_large_joint_angles(vd, cuda, omodels, wrap):
    """The ABA path's fp64 sin/cos (vd_sincos.cuh): Cody-Waite reduction for
    |q| ≤ 1e6, library fallback above.  Joint angles shifted by 2π·k must give
    the oracle's result on the same (shifted, rounded) inputs."""
    om = omodels["chain7"]
    m, dm = _dm(vd, "chain7")
    q, qd, _, tau = _states(om, 2048, 71)
    rng = np.random.default_rng(3)
    qs = q + 2 * np.pi * np.round(rng.uniform(-wrap, wrap, q.shape))
    ref, st = om.forward_dynamics(qs, qd, tau)
    got = _np(vd.forward_dynamics(dm, _t(qs), _t(qd), _t(tau)))
    cond = np.linalg.cond(om.crba(qs))
    assert np.all(rel_err(got, ref, axis=1) <= np.maximum(TOL64, 7 * np.finfo(np.float64).eps * cond))


@pytest.mark.parametrize("name,frame", [("chain7", "ee"), ("tree29", "l_palm"), ("tree29", "head")])
def test_osc_fp32(vd, cuda, omodels, name, frame):
    """fp32 osc_step (generated kernels for tree29) against the fp64 oracle:
    forward error bounded by ε₃₂·κ(M)·κ(J M⁻¹ Jᵀ + εI), flat 1e-4 where that
    product is small."""
    om = omodels[name]
    m, dm = _dm(vd, name)
    q, tau, lam, st, tau_ref, lam_ref, st_ref = _osc_case(vd, om, m, dm, name, 1024, 65, dtype=torch.float32,
                                                          frame=frame)
    ok = (st == 0) & (st_ref == 0)
    assert ok.mean() > 0.99
    kappa = np.linalg.cond(om.crba(q)) * np.linalg.cond(lam_ref)
    eps = np.finfo(np.float32).eps
    e_tau = rel_err(tau, tau_ref, axis=1)
    assert np.all(e_tau[ok] <= np.maximum(TOL32, om.n * eps * kappa[ok]))
    well = ok & (kappa * eps < 1e-6)
    assert e_tau[well].max(initial=0) <= TOL32


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("scale", [1.0, 3e3, 5e4])
def test_fp32_large_joint_angles(vd, cuda, omodels, generic, scale):
    """fp32 sin/cos of joint angles far outside [−π, π] (continuous joints
    wind up): vd_sincos_f32's Cody–Waite reduction below |q| = 1e4 and its
    sincosf fallback above, in the Panda ABA (generated, Cfg::kFast) and the
    loop kernels, against the oracle at the same float-rounded angles."""
    om = omodels["chain7"]
    m, dm = _dm(vd, "chain7", generic)
    q, qd, qdd, _ = _states(om, 4096, 71)
    wind = np.random.default_rng(3).integers(-1, 2, q.shape) * np.round(scale / (2 * np.pi)) * 2 * np.pi
    q32 = (q + wind).astype(np.float32).astype(np.float64)
    tau = om.rnea(q32, qd, qdd)
    got = _np(vd.rnea(dm, _t(q32, torch.float32), _t(qd, torch.float32), _t(qdd, torch.float32)))
    assert rel_err(got, tau, axis=1).max() <= TOL32
    a = _np(vd.forward_dynamics(dm, _t(q32, torch.float32), _t(qd, torch.float32), _t(tau, torch.float32)))
    _fd_check(om, q32, qd, tau, a, TOL32, "chain7")

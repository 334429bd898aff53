"""The generated straight-line robot routines (tools/gen_tree_kernels.py ->
vd_gen_robots.cuh), compiled for the host, against the oracle's LLT forward
dynamics (dynamics.hpp:421-444) and ABA restatement.  Runs without a GPU: it
checks the generator's symbolic algebra and structural-zero folding; the GPU
parity tests then check the same code on the device."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle_ffi import Model, rel_err

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2604_04310_b200", "csrc")


@pytest.fixture(scope="module")
def genlib(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("gen") / "gen_host.so")
    # FMA contraction as on the device (nvcc contracts mul+add by default)
    subprocess.run(["g++", "-O1", "-march=x86-64-v3", "-ffp-contract=fast", "-std=c++20", "-shared", "-fPIC", "-I", CSRC,
                    os.path.join(ROOT, "tests", "cpp", "gen_host.cpp"), "-o", so], check=True)
    L = ctypes.CDLL(so)
    L.gen_run_host.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long] + [ctypes.c_void_p] * 6
    return L


def _run(L, robot, op, xs, nout, g=(0.0, 0.0, 9.81), f32=False):
    """op: 0 aba, 1 rnea, 2 bias, 3 gravity, 4 crba, 5 fk (gen_host.cpp)."""
    dt = np.float32 if f32 else np.float64
    X = [np.asfortranarray(a.astype(dt)) for a in xs]
    N = X[0].shape[0]
    Y = np.zeros((N, nout), dtype=dt, order="F")
    st = np.zeros(N, dtype=np.int32)
    ptrs = [_p(a) for a in X] + [None] * (3 - len(X))
    ga = np.asarray(g, dtype=np.float64)
    bad = L.gen_run_host(robot, op, int(f32), N, *ptrs, _p(ga), _p(Y), _p(st))
    return Y.astype(np.float64), st, bad


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def test_generated_tables_are_current():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_tree_kernels.py"), "--check"],
                       capture_output=True, text=True)
    if "No such file" in r.stderr or "OSError" in r.stderr:
        pytest.skip("product library not built")
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("name,code", [("chain7", 1), ("tree29", 2)])
@pytest.mark.parametrize("f32", [False, True])
def test_generated_aba_matches_oracle(genlib, name, code, f32):
    om = Model.builtin(name)
    N = 2048
    q, qd, _, tau = om.random_states(N, 2604 + code, True, True)
    out, st, bad = _run(genlib, code, 0, (q, qd, tau), om.n, f32=f32)
    assert bad == 0
    ref, rst = om.forward_dynamics(q, qd, tau)
    assert np.all(rst == 0)
    err = rel_err(out.astype(np.float64), ref, axis=1)
    cond = np.linalg.cond(om.crba(q))
    # flat bar on well-conditioned states (DESIGN.md §Parity policy); the
    # fp32 G1 routine computes its floating-base trunk in fp64
    well = cond < 1e5
    tol = 1e-4 if f32 else 1e-10
    assert err[well].max(initial=0) <= tol
    # ill-conditioned instances (tree29 near base gimbal lock): forward-error
    # bound of a backward-stable solve, n·ε·κ(M) (DESIGN.md §Parity policy)
    eps = np.finfo(np.float32 if f32 else np.float64).eps
    bound = np.maximum(tol, om.n * eps * cond)
    assert np.all(err <= bound)


def test_generated_aba_with_gravity_roundtrip(genlib):
    """FD∘ID (test_dynamics.cpp:335-351) with non-standard gravity."""
    om = Model.builtin("tree29")
    N = 512
    q, qd, qdd, _ = om.random_states(N, 77, True, False)
    g = np.array([0.3, -0.4, 9.0])
    tau = om.rnea(q, qd, qdd, gravity=tuple(g))
    out, st, bad = _run(genlib, 2, 0, (q, qd, tau), om.n, g=g)
    assert bad == 0
    cosb = np.abs(np.cos(q[:, 4]))
    assert rel_err(out, qdd, axis=1)[cosb > 0.05].max() <= 1e-8


@pytest.mark.parametrize("name,code", [("chain7", 1), ("tree29", 2)])
@pytest.mark.parametrize("f32", [False, True])
def test_generated_rnea_family(genlib, name, code, f32):
    """rnea / bias / gravity (dynamics.hpp:222-267, 403-416, 434-435)."""
    om = Model.builtin(name)
    q, qd, qdd, _ = om.random_states(1024, 11 + code, True, False)
    tol = 1e-4 if f32 else 1e-10
    g = (0.3, -0.4, 9.0)
    got, _, _ = _run(genlib, code, 1, (q, qd, qdd), om.n, g=g, f32=f32)
    assert rel_err(got, om.rnea(q, qd, qdd, gravity=g), axis=1).max() <= tol
    z = np.zeros_like(q)
    got, _, _ = _run(genlib, code, 2, (q, qd), om.n, f32=f32)
    assert rel_err(got, om.rnea(q, qd, z), axis=1).max() <= tol
    got, _, _ = _run(genlib, code, 3, (q,), om.n, f32=f32)
    assert rel_err(got, om.rnea(q, z, z), axis=1).max() <= tol


@pytest.mark.parametrize("name,code", [("chain7", 1), ("tree29", 2)])
def test_generated_crba_and_fk(genlib, name, code):
    """crba (dynamics.hpp:337-365; exact zeros between branches) and
    forward_kinematics (kinematics.hpp:43-56)."""
    om = Model.builtin(name)
    n = om.n
    q, _, _, _ = om.random_states(1024, 21 + code, True, False)
    M, _, _ = _run(genlib, code, 4, (q,), n * n)
    ref = om.crba(q).transpose(0, 2, 1).reshape(len(q), -1)  # plane c·n + r = M(r, c)
    assert rel_err(M, ref, axis=1).max() <= 1e-10
    structural = np.all(ref == 0, axis=0)  # off-branch entries: zero for every state
    assert np.all(M[:, structural] == 0)  # exact zeros between branches, as in the reference
    F, _, _ = _run(genlib, code, 5, (q,), 12 * n)
    assert rel_err(F, om.fk(q).reshape(len(q), -1), axis=1).max() <= 1e-10


def _lower_pattern(om):
    """Branch-sparse lower triangle in compressed-column order, from the
    oracle's ancestor mask U (U[r, c] = 1 iff c is r or an ancestor of r)."""
    U = om.arrays()["mask"]
    return [(r, c) for c in range(om.n) for r in range(c, om.n) if U[r, c] != 0]


@pytest.mark.parametrize("name,code,nnz", [("chain7", 1, 28), ("tree29", 2, 242)])
@pytest.mark.parametrize("f32", [False, True])
def test_generated_packed_crba(genlib, name, code, nnz, f32):
    """The packed CRBA routine emits exactly the branch-sparse lower
    triangle of the reference's M (dynamics.hpp:331-350), and every entry it
    drops is an exact zero of the reference (test_dynamics.cpp:200-216)."""
    om = Model.builtin(name)
    pat = _lower_pattern(om)
    assert len(pat) == nnz
    q, _, _, _ = om.random_states(1024, 31 + code, True, False)
    Mp, _, _ = _run(genlib, code, 7, (q,), nnz, f32=f32)
    ref = om.crba(q)
    rows, cols = np.array(pat).T
    assert rel_err(Mp, ref[:, rows, cols], axis=1).max() <= (1e-4 if f32 else 1e-10)
    keep = np.zeros((om.n, om.n), bool)
    keep[rows, cols] = keep[cols, rows] = True
    assert np.all(ref[:, ~keep] == 0)
    if not f32:  # same generated arithmetic as the dense routine: bitwise equal
        Md, _, _ = _run(genlib, code, 4, (q,), om.n * om.n)
        assert np.array_equal(Mp, Md[:, cols * om.n + rows])


@pytest.mark.parametrize("name,code,frame", [("chain7", 1, "ee"), ("tree29", 2, "l_palm"), ("tree29", 2, "head"),
                                              ("tree29", 2, "r_foot")])
def test_generated_osc_matches_oracle(genlib, name, code, frame):
    """osc_step (control.hpp:108-155): τ and Λ against the oracle, with the
    conditioning-aware bound of test_gpu_parity.test_osc_fp64."""
    om = Model.builtin(name)
    N = 512
    q, qd, _, _ = om.random_states(N, 61, True, False)
    fid = {f[0]: f for f in om.frames()}[frame]
    fj, off = fid[1], fid[2]
    q0 = np.zeros((1, om.n))
    pose0, _ = om.jacobian(q0, frame)
    R0 = pose0[0, :9].reshape(3, 3, order="F")
    p0 = pose0[0, 9:]
    kp, kd, aff = [100.0] * 6, [20.0] * 6, [0.0] * 6
    posture = np.linspace(-0.3, 0.3, om.n)
    tau_ref, lam_ref, st_ref = om.osc(q, qd, frame, R0, p0, kp, kd, aff, posture, 10.0, 2.0)
    fR = off[:9].reshape(3, 3, order="F")  # frame offset, column-major R
    P = np.concatenate([fR.reshape(-1), off[9:], R0.reshape(-1), p0, kp, kd, aff, [10.0, 2.0, 1e-6], posture])
    genlib.gen_osc_host.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_long] + [ctypes.c_void_p] * 7
    Q, QD = np.asfortranarray(q), np.asfortranarray(qd)
    tau = np.zeros_like(Q, order="F")
    lam = np.zeros((N, 36), order="F")
    st = np.zeros(N, dtype=np.int32)
    g = np.array([0.0, 0.0, 9.81])
    bad = genlib.gen_osc_host(code, fj, N, _p(Q), _p(QD), _p(g), _p(P), _p(tau), _p(lam), _p(st))
    assert bad >= 0, "no generated variant for this frame joint"
    assert np.all(st == st_ref)
    ok = st == 0
    kappa = np.linalg.cond(om.crba(q)) * np.linalg.cond(lam_ref)
    bound = np.maximum(1e-10, 1e-16 * kappa)
    e_tau = rel_err(tau, tau_ref, axis=1)
    assert np.all(e_tau[ok] <= bound[ok]), float((e_tau / bound).max())
    e_lam = rel_err(lam, lam_ref.reshape(N, -1), axis=1)
    assert np.all(e_lam[ok] <= np.maximum(bound[ok], 1e-10)), float(e_lam.max())


@pytest.mark.parametrize("name,code", [("chain7", 1), ("tree29", 2)])
def test_generated_jvp_matches_oracle(genlib, name, code):
    """Generated dual-number ABA and RNEA against the oracle's Dual
    restatement (dual.hpp / autodiff.hpp): values and tangents."""
    om = Model.builtin(name)
    N = 512
    q, qd, qdd, tau = om.random_states(N, 81 + code, True, True)
    rng = np.random.default_rng(5)
    dq, dqd, dx2 = (rng.uniform(-1, 1, q.shape) for _ in range(3))
    genlib.gen_jvp_host.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_long] + [ctypes.c_void_p] * 10
    g = np.array([0.0, 0.0, 9.81])
    F = np.asfortranarray
    for op, x2, key in ((0, tau, "fd"), (1, qdd, "rnea")):
        X = [F(q), F(qd), F(x2)]
        DX = [F(dq), F(dqd), F(dx2)]
        y = np.zeros_like(X[0], order="F")
        dy = np.zeros_like(X[0], order="F")
        st = np.zeros(N, dtype=np.int32)
        bad = genlib.gen_jvp_host(code, op, N, *[_p(a) for a in X], *[_p(a) for a in DX], _p(g), _p(y), _p(dy), _p(st))
        assert bad == 0
        ref = om.jvp(key, (q, qd, x2), (dq, dqd, dx2))
        rv, rt = ref[0], ref[1]
        if key == "fd":
            cond = np.linalg.cond(om.crba(q))
            ok = cond < 1e5  # tangents of a solve inherit its conditioning twice
            assert rel_err(y, rv, axis=1)[ok].max() <= 1e-10
            assert rel_err(dy, rt, axis=1)[ok].max() <= 1e-9
        else:
            assert rel_err(y, rv, axis=1).max() <= 1e-10
            assert rel_err(dy, rt, axis=1).max() <= 1e-10


def test_generated_crba_fk_jvp_matches_oracle(genlib):
    """Generated dual-number CRBA and FK (tree29) against the oracle."""
    om = Model.builtin("tree29")
    N, n = 256, om.n
    q, _, _, _ = om.random_states(N, 91, True, False)
    dq = np.random.default_rng(6).uniform(-1, 1, q.shape)
    genlib.gen_jvp_host.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_long] + [ctypes.c_void_p] * 10
    g = np.array([0.0, 0.0, 9.81])
    Q, DQ = np.asfortranarray(q), np.asfortranarray(dq)
    for op, key, K in ((2, "crba", n * n), (3, "fk", 12 * n)):
        y = np.zeros((N, K), order="F")
        dy = np.zeros((N, K), order="F")
        st = np.zeros(N, dtype=np.int32)
        genlib.gen_jvp_host(2, op, N, _p(Q), None, None, _p(DQ), None, None, _p(g), _p(y), _p(dy), _p(st))
        rv, rt = om.jvp(key, (q,), (dq,))
        if key == "crba":
            rv, rt = (a.transpose(0, 2, 1).reshape(N, -1) for a in (rv, rt))
        else:
            rv, rt = rv.reshape(N, -1), rt.reshape(N, -1)
        assert rel_err(y, rv, axis=1).max() <= 1e-10
        assert rel_err(dy, rt, axis=1).max() <= 1e-10


@pytest.mark.parametrize("frame", ["l_palm", "head", "r_foot"])
def test_generated_task_routines_match_oracle(genlib, frame):
    """Generated Jacobian / diff-IK / manipulability (kinematics.hpp:89-153,
    control.hpp:79-97) for G1 task frames against the oracle."""
    om = Model.builtin("tree29")
    N = 512
    q, _, _, _ = om.random_states(N, 93, True, False)
    fid = {f[0]: f for f in om.frames()}[frame]
    fj, off = fid[1], fid[2]
    fR = off[:9].reshape(3, 3, order="F")
    q0 = np.zeros((1, om.n))
    pose0, _ = om.jacobian(q0, frame)
    R0, p0 = pose0[0, :9].reshape(3, 3, order="F"), pose0[0, 9:]
    kp, tw, damp = [2.0, 2.0, 2.0, 1.0, 1.0, 1.0], [0.1, 0.0, -0.1, 0.0, 0.2, 0.0], 0.05
    P = np.zeros(45 + om.n)
    P[:9], P[9:12], P[12:21], P[21:24] = fR.reshape(-1), off[9:], R0.reshape(-1), p0
    P[24:30], P[30:36], P[44] = kp, tw, damp
    genlib.gen_task_host.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_long] + [ctypes.c_void_p] * 6
    Q = np.asfortranarray(q)
    st = np.zeros(N, dtype=np.int32)
    pose = np.zeros((N, 12), order="F")
    J = np.zeros((N, 6 * om.n), order="F")
    assert genlib.gen_task_host(0, fj, N, _p(Q), _p(P), _p(pose), _p(J), _p(st), None) == 0
    rpose, rJ = om.jacobian(q, frame)
    assert rel_err(pose, rpose, axis=1).max() <= 1e-12
    assert rel_err(J, rJ.transpose(0, 2, 1).reshape(N, -1), axis=1).max() <= 1e-12  # plane 6 c + r
    qd = np.zeros((N, om.n), order="F")
    err = np.zeros((N, 6), order="F")
    assert genlib.gen_task_host(1, fj, N, _p(Q), _p(P), _p(qd), _p(err), _p(st), None) == 0
    rqd, rerr = om.diff_ik(q, frame, R0, p0, kp, tw, damp)
    assert rel_err(qd, rqd, axis=1).max() <= 1e-10
    assert rel_err(err, rerr, axis=1).max() <= 1e-10
    w = np.zeros((N, 1), order="F")
    assert genlib.gen_task_host(2, fj, N, _p(Q), _p(P), _p(w), None, _p(st), None) == 0
    assert rel_err(w[:, 0], om.manipulability(q, frame)) <= 1e-10
    # ManipJvp: the dual-number routine against the oracle's jvp_scalar, where
    # J Jᵀ is well conditioned (the derivative amplifies rounding by κ near a
    # singularity; tests/test_gpu_task.py states the bound)
    dq = np.asfortranarray(np.random.default_rng(4).standard_normal(q.shape))
    w2, dw = np.zeros((N, 1), order="F"), np.zeros((N, 1), order="F")
    assert genlib.gen_task_host(4, fj, N, _p(Q), _p(P), _p(w2), _p(dw), _p(st), _p(dq)) == 0
    rw, rdw = om.manipulability_jvp(q, dq, frame)
    assert rel_err(w2[:, 0], rw) <= 1e-10
    kappa = np.linalg.cond(np.einsum("nrk,nck->nrc", rJ, rJ))
    well = kappa < 1e3
    assert well.sum() > N // 4
    assert rel_err(dw[well, 0][:, None], rdw[well][:, None], axis=1).max() <= 1e-10


def _run_fext(L, robot, op, xs, fext, nout, g=(0.0, 0.0, 9.81), f32=False):
    """op: 8 rnea + f_ext, 9 bias + f_ext, 10 aba + f_ext (gen_host.cpp); fext (N, n, 6)."""
    dt = np.float32 if f32 else np.float64
    X = [np.asfortranarray(a.astype(dt)) for a in xs]
    N, n = X[0].shape
    F = np.asfortranarray(fext.reshape(N, 6 * n).astype(dt))  # plane 6 j + k
    Y = np.zeros((N, nout), dtype=dt, order="F")
    st = np.zeros(N, dtype=np.int32)
    ptrs = [_p(a) for a in X] + [None] * (3 - len(X))
    ga = np.asarray(g, dtype=np.float64)
    L.gen_run_fext_host.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long] + [ctypes.c_void_p] * 7
    bad = L.gen_run_fext_host(robot, op, int(f32), N, *ptrs, _p(F), _p(ga), _p(Y), _p(st))
    return Y.astype(np.float64), st, bad


@pytest.mark.parametrize("name,code", [("chain7", 1), ("tree29", 2)])
@pytest.mark.parametrize("f32", [False, True])
def test_generated_fext_routines_match_oracle(genlib, name, code, f32):
    """External wrenches (ExternalForcesT, dynamics.hpp:52-81, subtracted at
    243-245) in the generated RNEA, bias and ABA routines against the
    oracle on random world-frame wrenches and a non-standard gravity."""
    om = Model.builtin(name)
    N = 1024
    q, qd, qdd, tau = om.random_states(N, 4040 + code, True, True)
    rng = np.random.default_rng(7 + code)
    fext = rng.uniform(-5.0, 5.0, size=(N, om.n, 6))
    g = (0.2, -0.1, 9.5)
    tol = 1e-4 if f32 else 1e-10
    got, _, bad = _run_fext(genlib, code, 8, (q, qd, qdd), fext, om.n, g=g, f32=f32)
    assert bad == 0
    assert rel_err(got, om.rnea(q, qd, qdd, gravity=g, fext=fext), axis=1).max() <= tol
    got, _, _ = _run_fext(genlib, code, 9, (q, qd), fext, om.n, g=g, f32=f32)
    assert rel_err(got, om.rnea(q, qd, np.zeros_like(q), gravity=g, fext=fext), axis=1).max() <= tol
    got, st, bad = _run_fext(genlib, code, 10, (q, qd, tau), fext, om.n, g=g, f32=f32)
    assert bad == 0
    ref, rst = om.forward_dynamics(q, qd, tau, gravity=g, fext=fext)
    assert np.all(rst == 0)
    err = rel_err(got, ref, axis=1)
    cond = np.linalg.cond(om.crba(q))
    eps = np.finfo(np.float32 if f32 else np.float64).eps
    assert err[cond < 1e5].max(initial=0) <= tol
    assert np.all(err <= np.maximum(tol, om.n * eps * cond))


def test_generated_fused_dynamics(genlib):
    """GenChain7::Dyn (one prologue, CRBA + RNEA at q̈ = 0 + ABA) against the
    oracle's crba, rnea and LLT forward dynamics, and against the separately
    generated Crba / RneaBias / Aba routines on the same inputs."""
    om = Model.builtin("chain7")
    N, n = 1024, 7
    q, qd, _, tau = om.random_states(N, 88, True, True)
    F = lambda a: np.asfortranarray(a)  # noqa: E731
    M = np.zeros((N, n * n), order="F")
    b = np.zeros((N, n), order="F")
    a = np.zeros((N, n), order="F")
    st = np.zeros(N, dtype=np.int32)
    g = np.array([0.0, 0.0, 9.81])
    genlib.gen_dyn_host.argtypes = [ctypes.c_long] + [ctypes.c_void_p] * 8
    bad = genlib.gen_dyn_host(N, _p(F(q)), _p(F(qd)), _p(F(tau)), _p(g), _p(M), _p(b), _p(a), _p(st))
    assert bad == 0 and not st.any()
    Mo = M.reshape(N, n, n).transpose(0, 2, 1)  # plane c·n + r = M(r, c)
    assert rel_err(Mo, om.crba(q), axis=1).max() <= 1e-10
    assert rel_err(b, om.rnea(q, qd, np.zeros_like(q)), axis=1).max() <= 1e-10
    ref, _ = om.forward_dynamics(q, qd, tau)
    assert rel_err(a, ref, axis=1).max() <= 1e-10
    # the same expression graphs as the separate routines (up to FMA contraction)
    aba, _, _ = _run(genlib, 1, 0, [q, qd, tau], n)
    bias, _, _ = _run(genlib, 1, 2, [q, qd], n)
    crba, _, _ = _run(genlib, 1, 4, [q], n * n)
    assert rel_err(a, aba, axis=1).max() <= 1e-13
    assert rel_err(b, bias, axis=1).max() <= 1e-13
    assert rel_err(M, crba, axis=1).max() <= 1e-13

"""Pins the oracle's forward-mode JVPs (oracle/orc_dual.hpp restating
dual.hpp:14-180, run through the oracle's scalar-generic algorithms like
autodiff.hpp:41-52).  The reference ships no JVP tests or golden vectors; its
SPEC states the acceptance properties: JVPs of rnea
and crba w.r.t. (q, q̇, q̈) match central finite differences with step 1e-6 to
1e-5 relative, and are linear in the tangent to 1e-12.  Those are checked
here on CPU, for the vectorized and the loop forms, plus FK and forward
dynamics, and the dual values equal the plain double evaluation."""
import numpy as np
import pytest

from oracle_ffi import Model as OModel
from oracle_ffi import rel_err

ROBOTS = ["chain7", "tree29", "humanoid23"]


@pytest.fixture(scope="module")
def models(oracle):
    return {n: OModel.builtin(n) for n in ROBOTS}


def _fd(f, x, v, h=1e-6):
    return (f(x + h * v) - f(x - h * v)) / (2 * h)


def _case(om, N, seed):
    q, qd, qdd, tau = om.random_states(N, seed, True, True)
    rng = np.random.default_rng(seed)
    return q, qd, qdd, tau, [rng.standard_normal(q.shape) for _ in range(3)]


@pytest.mark.parametrize("name", ROBOTS)
@pytest.mark.parametrize("variant", [0, 1])
def test_rnea_jvp_matches_finite_differences(models, name, variant):
    om = models[name]
    q, qd, qdd, _, (vq, vqd, vqdd) = _case(om, 100, 1)
    loop = bool(variant)
    val, tan = om.jvp("rnea", (q, qd, qdd), (vq, vqd, vqdd), variant=variant)
    assert rel_err(val, om.rnea(q, qd, qdd, loop=loop), axis=1).max() <= 1e-14
    fd = (_fd(lambda x: om.rnea(x, qd, qdd, loop=loop), q, vq) + _fd(lambda x: om.rnea(q, x, qdd, loop=loop), qd, vqd)
          + _fd(lambda x: om.rnea(q, qd, x, loop=loop), qdd, vqdd))
    assert rel_err(tan, fd, axis=1).max() <= 1e-5


@pytest.mark.parametrize("name", ROBOTS)
@pytest.mark.parametrize("variant", [0, 1])
def test_crba_jvp_matches_finite_differences(models, name, variant):
    om = models[name]
    q, _, _, _, (vq, _, _) = _case(om, 100, 2)
    val, tan = om.jvp("crba", (q,), (vq,), variant=variant)
    assert rel_err(val, om.crba(q), axis=1).max() <= 1e-14
    fd = _fd(lambda x: om.crba(x), q, vq)
    assert rel_err(tan, fd, axis=1).max() <= 1e-5


@pytest.mark.parametrize("name", ROBOTS)
def test_fk_and_fd_jvp_match_finite_differences(models, name):
    om = models[name]
    q, qd, _, tau, (vq, vqd, vtau) = _case(om, 100, 3)
    val, tan = om.jvp("fk", (q,), (vq,))
    fk = lambda x: om.fk(x).reshape(x.shape[0], -1)  # noqa: E731
    assert rel_err(val, fk(q), axis=1).max() <= 1e-14
    assert rel_err(tan, _fd(fk, q, vq), axis=1).max() <= 1e-5
    for variant in (0, 1):
        aba = bool(variant)
        val, tan, st = om.jvp("fd", (q, qd, tau), (vq, vqd, vtau), variant=variant)
        assert np.all(st == 0)
        f = lambda a, b, c: om.forward_dynamics(a, b, c, aba=aba)[0]  # noqa: E731
        fd = _fd(lambda x: f(x, qd, tau), q, vq) + _fd(lambda x: f(q, x, tau), qd, vqd) + _fd(
            lambda x: f(q, qd, x), tau, vtau)
        # forward dynamics amplifies by κ(M); compare per instance with the
        # finite-difference truncation/roundoff floor scaled likewise
        cond = np.linalg.cond(om.crba(q))
        e = rel_err(tan, fd, axis=1)
        assert np.all(e <= np.maximum(1e-5, 1e-9 * cond)), float(e.max())


@pytest.mark.parametrize("name", ["chain7", "tree29"])
def test_jvp_is_linear_in_tangent(models, name):
    om = models[name]
    q, qd, qdd, _, (v1, v2, v3) = _case(om, 50, 4)
    a, b = 0.7, -1.3
    _, t1 = om.jvp("rnea", (q, qd, qdd), (v1, v2, v3))
    _, t2 = om.jvp("rnea", (q, qd, qdd), (v3, v1, v2))
    _, t12 = om.jvp("rnea", (q, qd, qdd), (a * v1 + b * v3, a * v2 + b * v1, a * v3 + b * v2))
    assert rel_err(t12, a * t1 + b * t2, axis=1).max() <= 1e-12
    _, m1 = om.jvp("crba", (q,), (v1,))
    _, m2 = om.jvp("crba", (q,), (v2,))
    _, m12 = om.jvp("crba", (q,), (a * v1 + b * v2,))
    assert rel_err(m12, a * m1 + b * m2, axis=1).max() <= 1e-12


def test_vectorized_and_loop_jvps_agree(models):
    om = models["tree29"]
    q, qd, qdd, _, (vq, vqd, vqdd) = _case(om, 200, 5)
    _, t0 = om.jvp("rnea", (q, qd, qdd), (vq, vqd, vqdd), variant=0)
    _, t1 = om.jvp("rnea", (q, qd, qdd), (vq, vqd, vqdd), variant=1)
    assert rel_err(t0, t1, axis=1).max() <= 1e-12
    _, m0 = om.jvp("crba", (q,), (vq,), variant=0)
    _, m1 = om.jvp("crba", (q,), (vq,), variant=1)
    assert rel_err(m0, m1, axis=1).max() <= 1e-12


def test_jvp_qd_direction_is_coriolis_derivative(models):
    """jvp(rnea) along q̇ at q̈ = 0 equals the directional derivative
    of the Coriolis vector (gravity does not depend on q̇)."""
    om = models["chain7"]
    q, qd, _, _, (_, v, _) = _case(om, 50, 6)
    z = np.zeros_like(q)
    _, t = om.jvp("rnea", (q, qd, z), (None, v, None))
    fd = _fd(lambda x: om.rnea(q, x, z, gravity=(0, 0, 0)), qd, v)
    assert rel_err(t, fd, axis=1).max() <= 1e-5

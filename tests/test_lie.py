"""lie_derivative (control.hpp:157-163) and the manipulability JVP it takes for
the SPEC's CBF example, on CPU:

* the oracle's dual-number manipulability JVP (orc_batch_manip_jvp, jvp_scalar
  of kinematics.hpp:138-153) against central finite differences of its own
  manipulability, and its value against the plain evaluation — this pins the
  checker the GPU tests use;
* the SPEC example h = manipulability ∘ J(q), f = forward-dynamics drift:
  L_f h equals the finite-difference directional derivative to 1e-4;
* the batched Python combinator on the SPEC's analytic examples (h constant
  → 0; h = ½‖z‖², f = z → ‖z‖²) and its dimension check, with torch CPU
  tensors (it is pure composition: no kernel of its own)."""
import numpy as np
import pytest
import torch

from oracle_ffi import Model as OModel

FRAMES = {"chain7": "ee", "tree29": "l_palm", "humanoid23": "l_palm"}


@pytest.fixture(scope="module")
def models(oracle):
    return {n: OModel.builtin(n) for n in FRAMES}


@pytest.mark.parametrize("name", list(FRAMES))
def test_oracle_manip_jvp_matches_finite_differences(models, name):
    om = models[name]
    frame = FRAMES[name]
    q, qd, _, _ = om.random_states(64, 77, True, False)
    v = np.random.default_rng(1).standard_normal(q.shape)
    w, dw = om.manipulability_jvp(q, v, frame)
    assert np.abs(w - om.manipulability(q, frame)).max() <= 1e-13  # the same arithmetic on dual values
    h = 1e-6
    fd = (om.manipulability(q + h * v, frame) - om.manipulability(q - h * v, frame)) / (2 * h)
    ok = w > 1e-4  # away from singular configurations, where w is not differentiable
    assert ok.sum() > 32
    assert np.all(np.abs(dw - fd)[ok] <= 1e-6 * np.maximum(1.0, np.abs(fd[ok])))
    # linear in the tangent
    _, dw2 = om.manipulability_jvp(q, 2.5 * v - qd, frame)
    _, dwq = om.manipulability_jvp(q, qd, frame)
    assert np.allclose(dw2[ok], (2.5 * dw - dwq)[ok], rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("name", ["chain7", "tree29"])
def test_spec_example_manipulability_along_dynamics_drift(models, name):
    """h = manipulability ∘ J(q), f = FD drift (q̇, q̈(q, q̇, τ = 0)):
    L_f h matches the finite-difference directional derivative, rel tol 1e-4."""
    om = models[name]
    frame = FRAMES[name]
    q, qd, _, _ = om.random_states(32, 78, True, False)
    qdd, st = om.forward_dynamics(q, qd, np.zeros_like(q))
    assert np.all(st == 0)
    # z = (q, q̇); f(z) = (q̇, q̈); h depends on q only, so L_f h = JVP along q̇
    _, lie = om.manipulability_jvp(q, qd, frame)
    h = 1e-6
    fd = (om.manipulability(q + h * qd, frame) - om.manipulability(q - h * qd, frame)) / (2 * h)
    w = om.manipulability(q, frame)
    ok = w > 1e-4
    assert np.all(np.abs(lie - fd)[ok] <= 1e-4 * np.maximum(np.abs(fd[ok]), 1e-3))
    del qdd


def test_lie_derivative_combinator_spec_examples(vd):
    z = torch.randn(1000, 14, dtype=torch.float64, generator=torch.Generator().manual_seed(3))
    # h constant -> 0
    const = lambda z, dz: (torch.full((z.shape[0],), 4.0, dtype=z.dtype), torch.zeros(z.shape[0], dtype=z.dtype))  # noqa: E731
    assert torch.equal(vd.lie_derivative(const, lambda z: torch.sin(z), z), torch.zeros(1000, dtype=torch.float64))
    # h = ½‖z‖², f = z -> ‖z‖²
    half_sq = lambda z, dz: (0.5 * (z * z).sum(1), (z * dz).sum(1))  # noqa: E731
    got = vd.lie_derivative(half_sq, lambda z: z, z)
    assert torch.allclose(got, (z * z).sum(1), rtol=1e-15, atol=0)
    # f(z) must have z's shape (DimensionError, autodiff.hpp:56-59)
    with pytest.raises(vd.DimensionError):
        vd.lie_derivative(half_sq, lambda z: z[:, :7], z)


def test_jvp_combinators(vd):
    """jvp / jvp_scalar / jacobian_fwd (autodiff.hpp:41-84) on a torch JVP:
    h(x) = (x0 x1, sin x2) has the Jacobian [[x1, x0, 0], [0, 0, cos x2]]."""
    x = torch.randn(64, 3, dtype=torch.float64, generator=torch.Generator().manual_seed(5))

    def h(x, dx):
        val = torch.stack([x[:, 0] * x[:, 1], torch.sin(x[:, 2])], 1)
        tan = torch.stack([dx[:, 0] * x[:, 1] + x[:, 0] * dx[:, 1], torch.cos(x[:, 2]) * dx[:, 2]], 1)
        return val, tan

    J = vd.jacobian_fwd(h, x)
    ref = torch.zeros(64, 2, 3, dtype=torch.float64)
    ref[:, 0, 0], ref[:, 0, 1], ref[:, 1, 2] = x[:, 1], x[:, 0], torch.cos(x[:, 2])
    assert torch.equal(J, ref)
    v = torch.randn(64, 3, dtype=torch.float64)
    assert torch.allclose(vd.jvp(h, x, v)[1], torch.einsum("nij,nj->ni", J, v), rtol=1e-15, atol=1e-15)
    with pytest.raises(vd.DimensionError):
        vd.jvp(h, x, v[:, :2])
    with pytest.raises(vd.DimensionError):
        vd.jvp_scalar(h, x, v)
    s = lambda x, dx: (h(x, dx)[0][:, 0], h(x, dx)[1][:, 0])  # noqa: E731
    assert torch.equal(vd.jvp_scalar(s, x, v)[1], h(x, v)[1][:, 0])

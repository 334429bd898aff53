"""vd_rows_to_planes / vd_planes_to_rows: row-major batch <-> the planes the
kernels read (batch.hpp:15-19 column-major StateBatch), bitwise, with
ragged N, leading dimensions beyond the data and rows wider than one CTA's
staging tile."""
import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K", [1, 2, 7, 29, 42, 174, 385])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_rows_planes_roundtrip(vd, cuda, K, dtype):
    lib = vd._lib.load()
    code = 0 if dtype == torch.float64 else 1
    for N in (1, 33, 1001, 70001):
        ldr, ldp = K + 3, N + 5
        rows = torch.randn((N, ldr), dtype=torch.float64, device="cuda").to(dtype)
        planes = torch.full((K, ldp), float("nan"), dtype=dtype, device="cuda")
        p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        assert lib.vd_rows_to_planes(code, N, K, p(rows), ldr, p(planes), ldp, None) == 0
        torch.cuda.synchronize()
        assert torch.equal(planes[:, :N], rows[:, :K].t())
        assert torch.isnan(planes[:, N:]).all()
        back = torch.full((N, ldr), float("nan"), dtype=dtype, device="cuda")
        assert lib.vd_planes_to_rows(code, N, K, p(planes), ldp, p(back), ldr, None) == 0
        torch.cuda.synchronize()
        assert torch.equal(back[:, :K], rows[:, :K])
        assert torch.isnan(back[:, K:]).all()
    # argument checks
    assert lib.vd_rows_to_planes(code, 10, K, p(rows), K - 1 if K > 1 else 0, p(planes), 10, None) != 0
    assert lib.vd_rows_to_planes(code, 0, K, None, 0, None, 0, None) == 0


def test_python_api_row_major_inputs(vd, cuda):
    """Row-major (N, n) inputs through the staged transpose give bitwise the
    result of column-major (already plane-layout) inputs."""
    m = vd.robots.tree29()
    dm = vd.DeviceModel(m, 0)
    N, n = 5000, m.dof()
    x = [torch.rand((N, n), dtype=torch.float64, device="cuda") for _ in range(3)]
    xc = [t.t().contiguous().t() for t in x]  # same values, column-major
    assert torch.equal(vd.rnea(dm, *x), vd.rnea(dm, *xc))
    f = torch.rand((N, n, 6), dtype=torch.float64, device="cuda")
    assert torch.equal(vd.forward_dynamics(dm, *x, fext=f), vd.forward_dynamics(dm, *xc, fext=f.clone()))

"""Per-model JIT modules (paper_2604_04310_b200/jit.py) without a GPU: the
generated translation unit compiles for sm_100a, exports exactly the vdj_*
entry points, attaches to its own model and is refused by any other
(fingerprint check)."""
import subprocess

import pytest

from urdf_gen import random_urdf


@pytest.fixture(scope="module")
def jitmod(vd):
    from paper_2604_04310_b200 import jit

    m = vd.urdf.load_model_from_string(random_urdf(5, n=12))
    return m, jit.build(m)


def test_jit_module_exports(jitmod):
    _, path = jitmod
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    syms = sorted(ln.split()[-1] for ln in out.splitlines() if ln.split() and ln.split()[-1].startswith("vdj_"))
    assert syms == ["vdj_abi_version", "vdj_dof", "vdj_fingerprint", "vdj_init", "vdj_launch"]
    # nothing of the launch machinery leaks (-fvisibility=hidden)
    assert "scratch_alloc" not in out


def test_jit_attach_checks_the_model(vd, jitmod):
    from paper_2604_04310_b200 import jit

    m, path = jitmod
    assert jit.attach(m, path) == path
    other = vd.urdf.load_model_from_string(random_urdf(6, n=12))
    with pytest.raises(RuntimeError, match="another model"):
        jit.attach(other, path)
    lib = vd._lib.load()
    assert lib.vd_model_attach_jit(m.handle, b"/nonexistent/vdj.so") != 0


def test_jit_cache_is_reused(vd, jitmod):
    from paper_2604_04310_b200 import jit

    m, path = jitmod
    assert jit.build(m) == path  # same model, same source: the cached module


def test_jit_skips_models_without_joints(vd):
    from paper_2604_04310_b200 import jit

    text = ('<robot name="empty"><link name="base"><inertial><mass value="1.0"/>'
            '<inertia ixx="1" ixy="0" ixz="0" iyy="1" iyz="0" izz="1"/></inertial></link></robot>')
    m = vd.urdf.load_model_from_string(text)
    assert m.dof() == 0
    assert jit.attach(m) is None

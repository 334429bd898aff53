"""CPU-side checks of the drop-in boundary (no GPU needed):

* libvecdyn_cuda.so loads and exports every symbol include/vecdyn_cuda.h declares;
* the host model layer (URDF reader, builder, floating base, packer) produces
  the same RobotModel as the oracle's restatement of proj/core/src/*.cpp on the
  builtin robots and on random URDF documents;
* error codes mirror the reference exception types (errors.hpp:9-61);
* random_states is bit-identical to the reference's mt19937_64 stream;
* compute entry points fail loudly (VD_ERR_CUDA) without a GPU instead of
  falling back to the CPU.
"""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle_ffi import Model as OModel
from urdf_gen import random_urdf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vecdyn_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vd_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported(vd):
    lib = ctypes.CDLL(vd._lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding types every one of them
    assert set(syms) <= set(vd._lib.SIGNATURES)


def _same_model(vm, om, tol=1e-15):
    n = om.n
    assert vm.dof() == n
    a = om.arrays()
    assert vm.parents() == list(a["parent"])
    assert vm.joint_names() == om.joint_names()
    for i in range(n):
        t, ax, off, I = vm.joint(i)
        assert t == a["type"][i]
        assert np.abs(ax - a["axis"][i]).max() <= 4e-16  # axis / |axis| (model.cpp:319-326), ulp-level
        R = off[:9].reshape(3, 3, order="F")
        Ro = a["offset"][i][:9].reshape(3, 3)
        assert np.abs(R - Ro).max() <= tol
        assert np.abs(off[9:] - a["offset"][i][9:]).max() <= tol
        scale = max(1.0, np.abs(a["inertia"][i]).max())
        assert np.abs(I - a["inertia"][i]).max() <= tol * scale * 10
    assert np.array_equal(vm.ancestor_mask(), a["mask"])
    vf, of = vm.frames(), om.frames()
    assert [(f[0], f[1]) for f in vf] == [(f[0], f[1]) for f in of]
    for (nm, j, off), (_, _, ooff) in zip(vf, of):
        assert np.abs(off[:9].reshape(3, 3, order="F") - ooff[:9].reshape(3, 3)).max() <= tol
        assert np.abs(off[9:] - ooff[9:]).max() <= tol


@pytest.mark.parametrize("name", ["chain7", "humanoid23", "tree29"])
def test_builtin_models_match_oracle(vd, oracle, name):
    vm = vd.robots.by_name(name)
    om = OModel.builtin(name)
    _same_model(vm, om)
    assert vm.total_mass() == pytest.approx(om.total_mass(), rel=1e-15)
    assert vm.is_serial_chain() == (name == "chain7")
    facts = {"chain7": (7, 7), "humanoid23": (23, 6), "tree29": (29, 12)}[name]
    assert (vm.dof(), vm.max_depth()) == facts


def test_robot_facts(vd):
    """SURVEY §3.1 / Appendix A facts about the two benchmark robots."""
    t = vd.robots.tree29()
    names = t.joint_names()
    assert names[:6] == ["base_tx", "base_ty", "base_tz", "base_rz", "base_ry", "base_rx"]
    assert names[6] == "l_hip_yaw" and names[18] == "waist_yaw" and names[19] == "l_shoulder_pitch"
    assert int(t.ancestor_mask().sum()) == 242
    assert t.total_mass() == pytest.approx(34.0)
    assert len(t.warnings()) >= 1  # massless floating stack flagged (model.cpp:277-285)
    c = vd.robots.chain7()
    assert c.total_mass() == pytest.approx(15.07)
    frames = {f[0]: f for f in c.frames()}
    assert frames["ee"][1] == 6 and np.allclose(frames["ee"][2][9:], [0, 0, 0.107])


@pytest.mark.parametrize("seed", range(8))
def test_random_urdf_models_match_oracle(vd, oracle, seed):
    text = random_urdf(seed, n=14, branchiness=0.6)
    _same_model(vd.urdf.load_model_from_string(text), OModel.from_urdf(text), tol=1e-14)


def test_floating_base_matches_oracle(vd, oracle):
    text = random_urdf(99, n=6)
    fm = vd.floating_base(vd.urdf.load_model_from_string(text))
    om = OModel.from_urdf(text).floating()
    _same_model(fm, om, tol=1e-14)


BAD_DOCS = [
    ("<a>\n  <b>\n  </c>\n</a>", 2, (3, 3)),                       # mismatched tag (test_urdf.cpp:103-111)
    ("<a><b></b>", 2, None),                                        # unterminated
    ('<a x="&bogus;"/>', 2, None),                                  # bad entity
    ("<!DOCTYPE robot><robot/>", 2, None),                          # doctype rejected
    ('<a x="1" x="2"/>', 2, None),                                  # duplicate attribute
    ("<notrobot/>", 2, None),
    ('<robot name="c"><link name="a"/><link name="b"/>'
     '<joint name="j1" type="fixed"><parent link="a"/><child link="b"/></joint>'
     '<joint name="j2" type="fixed"><parent link="b"/><child link="a"/></joint></robot>', 3, None),  # cycle
    ('<robot name="d"><link name="a"/>'
     '<joint name="j" type="fixed"><parent link="a"/><child link="ghost"/></joint></robot>', 3, None),
    ('<robot name="p"><link name="a"/><link name="b"/>'
     '<joint name="j" type="planar"><parent link="a"/><child link="b"/></joint></robot>', 5, None),
    ('<robot name="m"><link name="base"/><link name="mid"/>'
     '<link name="tip"><inertial><mass value="1"/><inertia ixx="0.1" ixy="0" ixz="0" iyy="0.1" iyz="0" izz="0.1"/>'
     '</inertial></link>'
     '<joint name="j1" type="revolute"><parent link="base"/><child link="mid"/><axis xyz="0 1 0"/></joint>'
     '<joint name="j2" type="revolute"><parent link="mid"/><child link="tip"/><axis xyz="0 1 0"/></joint></robot>',
     3, None),                                                      # missing inertial names the link
    ('<robot name="x"><link name="a"/><link name="b"><inertial><mass value="abc"/>'
     '<inertia ixx="1" ixy="0" ixz="0" iyy="1" iyz="0" izz="1"/></inertial></link>'
     '<joint name="j" type="revolute"><parent link="a"/><child link="b"/></joint></robot>', 2, None),
    ('<robot name="x"><link name="a"/><link name="b"><inertial><mass value="1"/>'
     '<inertia ixx="1" ixy="0" ixz="0" iyy="1" iyz="0" izz="1"/></inertial></link>'
     '<joint name="j" type="revolute"><parent link="a"/><child link="b"/><axis xyz="0 0 2"/></joint></robot>',
     3, None),                                                      # non-unit axis
]


@pytest.mark.parametrize("doc,code,pos", BAD_DOCS)
def test_error_codes_match_oracle(vd, oracle, doc, code, pos):
    lib = vd._lib.load()
    h = ctypes.c_void_p()
    data = doc.encode()
    rc = lib.vd_model_load_urdf_string(data, len(data), ctypes.byref(h))
    assert rc == code, lib.vd_last_error()
    with pytest.raises(oracle.OracleError) as ei:
        OModel.from_urdf(doc)
    assert ei.value.code == code
    if pos:
        assert (lib.vd_last_error_line(), lib.vd_last_error_column()) == pos
    if "mid" in doc:
        assert b"mid" in lib.vd_last_error()


def test_python_exceptions(vd):
    with pytest.raises(vd.ParseError) as ei:
        vd.urdf.load_model_from_string("<a>\n  <b>\n  </c>\n</a>")
    assert (ei.value.line, ei.value.column) == (3, 3)
    with pytest.raises(vd.UnknownFrameError):
        vd.robots.chain7().frame_index("nope")
    with pytest.raises(vd.Error):
        vd.robots.by_name("nope")
    with pytest.raises(vd.Error):
        vd.urdf.load_model("/nonexistent.urdf")


def test_random_states_bit_identical(vd, oracle):
    for name in ("chain7", "tree29"):
        vm, om = vd.robots.by_name(name), OModel.builtin(name)
        b = vd.random_states(vm, 777, 2604, True, True)
        q, qd, qdd, tau = om.random_states(777, 2604, True, True)
        for x, y in ((b.q, q), (b.qd, qd), (b.qdd, qdd), (b.tau, tau)):
            assert np.array_equal(x, y)
        b2 = vd.random_states(vm, 5, 1, False, False)
        assert b2.qdd is None and b2.tau is None


def test_shard_ranges(vd):
    for N in (0, 1, 7, 4096, 4194304, 1000003):
        for W in (1, 2, 3, 4, 8):
            spans = [vd.shard_range(N, W, r) for r in range(W)]
            assert spans[0][0] == 0 and spans[-1][1] == N
            for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
                assert e0 == b1
            assert sum(e - b for b, e in spans) == N


def test_no_cpu_fallback_without_gpu(vd):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present; covered by the gpu suite")
    m = vd.robots.chain7()
    with pytest.raises(vd.CudaError):
        vd.DeviceModel(m, 0)
    lib = vd._lib.load()
    q = np.zeros((4, 7), order="F")
    out = np.zeros((4, 7), order="F")
    rc = lib.vd_batch_rnea_host(m.handle, 4, q.ctypes.data, q.ctypes.data, q.ctypes.data, None, out.ctypes.data,
                                None, 0)
    assert rc == vd._lib.VD_ERR_CUDA


def test_robot_tables_current(vd):
    """The committed compile-time robot tables match what the packer produces."""
    import subprocess
    import sys

    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_robot_tables.py"), "--check"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr

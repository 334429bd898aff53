"""ctypes binding of the CPU oracle (oracle/build/liborc.so) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this
module.  All batch functions use the reference's column-major SoA layout:
element (i, k) at k*N + i, exposed here as numpy arrays shaped (N, K) with
Fortran order.
"""
import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB = os.path.join(ORACLE_DIR, "build", "liborc.so")
PORT_TESTS = os.path.join(ORACLE_DIR, "build", "orc_port_tests")

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", ORACLE_DIR, "-j8"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        vp, i64, ci, cd, cc = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_char_p
        L.orc_last_error.restype = cc
        L.orc_model_builtin.restype = vp
        L.orc_model_builtin.argtypes = [cc]
        L.orc_model_from_urdf.restype = vp
        L.orc_model_from_urdf.argtypes = [cc]
        L.orc_model_from_urdf_status.argtypes = [cc, ctypes.POINTER(vp)]
        L.orc_model_floating.restype = vp
        L.orc_model_floating.argtypes = [vp]
        L.orc_model_free.argtypes = [vp]
        for f in ("orc_model_dof", "orc_model_max_depth", "orc_model_is_serial", "orc_model_warning_count",
                  "orc_model_frame_count"):
            getattr(L, f).argtypes = [vp]
        L.orc_model_total_mass.restype = cd
        L.orc_model_total_mass.argtypes = [vp]
        L.orc_model_arrays.argtypes = [vp] + [vp] * 6
        L.orc_model_joint_name.argtypes = [vp, ci, ctypes.c_char_p, ci]
        L.orc_model_frame.argtypes = [vp, ci, ctypes.c_char_p, ci, ctypes.POINTER(ci), vp]
        L.orc_frame_id.argtypes = [vp, cc]
        L.orc_random_states.argtypes = [vp, i64, ctypes.c_uint64, vp, vp, vp, vp]
        L.orc_batch_rnea.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, ci, ci, ci]
        L.orc_batch_crba.argtypes = [vp, i64, vp, vp, ci, ci, ci]
        L.orc_batch_fd.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, vp, ci, ci]
        L.orc_batch_fk.argtypes = [vp, i64, vp, vp, ci, ci]
        L.orc_batch_jacobian.argtypes = [vp, i64, vp, cc, vp, vp, ci]
        L.orc_batch_osc.argtypes = [vp, i64, vp, vp, cc, vp, vp, vp, vp, vp, cd, cd, vp, cd, vp, vp, vp, ci]
        L.orc_batch_diffik.argtypes = [vp, i64, vp, cc, vp, vp, vp, cd, vp, vp, ci]
        L.orc_batch_manip.argtypes = [vp, i64, vp, cc, vp, ci]
        L.orc_batch_manip_jvp.argtypes = [vp, i64, vp, vp, cc, vp, vp, ci]
        L.orc_batch_jvp.argtypes = [vp, ci, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, ci, ci]
        _lib = L
    return _lib


def _ptr(a):
    return ctypes.c_void_p(0 if a is None else a.ctypes.data)


def _F(a):
    return None if a is None else np.asfortranarray(np.asarray(a, dtype=np.float64))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _chk(rc):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


class Model:
    def __init__(self, handle):
        if not handle:
            raise OracleError(-1, lib().orc_last_error().decode())
        self.h = ctypes.c_void_p(handle)

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and _lib is not None:
            _lib.orc_model_free(self.h)

    @staticmethod
    def builtin(name):
        return Model(lib().orc_model_builtin(name.encode()))

    @staticmethod
    def from_urdf(text):
        h = ctypes.c_void_p()
        rc = lib().orc_model_from_urdf_status(text.encode(), ctypes.byref(h))
        if rc:
            raise OracleError(rc, lib().orc_last_error().decode())
        return Model(h.value)

    def floating(self):
        return Model(lib().orc_model_floating(self.h))

    @property
    def n(self):
        return lib().orc_model_dof(self.h)

    def total_mass(self):
        return lib().orc_model_total_mass(self.h)

    def arrays(self):
        n = self.n
        par = np.zeros(n, dtype=np.int32)
        typ = np.zeros(n, dtype=np.int32)
        ax = np.zeros((n, 3))
        off = np.zeros((n, 12))
        ine = np.zeros((n, 36))
        mask = np.zeros((n, n))
        lib().orc_model_arrays(self.h, _ptr(par), _ptr(typ), _ptr(ax), _ptr(off), _ptr(ine), _ptr(mask))
        return dict(parent=par, type=typ, axis=ax, offset=off, inertia=ine.reshape(n, 6, 6), mask=mask)

    def joint_names(self):
        out = []
        for i in range(self.n):
            b = ctypes.create_string_buffer(256)
            lib().orc_model_joint_name(self.h, i, b, 256)
            out.append(b.value.decode())
        return out

    def frames(self):
        out = []
        for k in range(lib().orc_model_frame_count(self.h)):
            b = ctypes.create_string_buffer(256)
            j = ctypes.c_int()
            off = np.zeros(12)
            lib().orc_model_frame(self.h, k, b, 256, ctypes.byref(j), _ptr(off))
            out.append((b.value.decode(), j.value, off))
        return out

    def frame_id(self, name):
        return lib().orc_frame_id(self.h, name.encode())

    # ---------------------------------------------------------------- batch evaluation
    def random_states(self, N, seed, with_qdd=True, with_tau=False):
        n = self.n
        q, qd = np.empty((N, n), order="F"), np.empty((N, n), order="F")
        qdd = np.empty((N, n), order="F") if with_qdd else None
        tau = np.empty((N, n), order="F") if with_tau else None
        lib().orc_random_states(self.h, N, seed, _ptr(q), _ptr(qd), _ptr(qdd), _ptr(tau))
        return q, qd, qdd, tau

    def rnea(self, q, qd, qdd, gravity=(0, 0, 9.81), fext=None, threads=0, loop=False, f32=False):
        q, qd, qdd = _F(q), _F(qd), _F(qdd)
        N = q.shape[0]
        g = np.asarray(gravity, dtype=np.float64)
        fx = None if fext is None else np.asfortranarray(np.asarray(fext, dtype=np.float64).reshape(N, -1))
        out = np.empty((N, self.n), order="F")
        _chk(lib().orc_batch_rnea(self.h, N, _ptr(q), _ptr(qd), _ptr(qdd), _ptr(g), _ptr(fx), _ptr(out), threads,
                                  1 if loop else 0, 1 if f32 else 0))
        return out

    def crba(self, q, threads=0, loop=False, f32=False):
        q = _F(q)
        N, n = q.shape[0], self.n
        out = np.empty((N, n * n), order="F")
        _chk(lib().orc_batch_crba(self.h, N, _ptr(q), _ptr(out), threads, 1 if loop else 0, 1 if f32 else 0))
        return out.reshape(N, n, n, order="C").transpose(0, 2, 1)  # M[i] = column-major n x n

    def forward_dynamics(self, q, qd, tau, gravity=(0, 0, 9.81), fext=None, threads=0, aba=False):
        q, qd, tau = _F(q), _F(qd), _F(tau)
        N = q.shape[0]
        g = np.asarray(gravity, dtype=np.float64)
        fx = None if fext is None else np.asfortranarray(np.asarray(fext, dtype=np.float64).reshape(N, -1))
        out = np.empty((N, self.n), order="F")
        st = np.zeros(N, dtype=np.int32)
        _chk(lib().orc_batch_fd(self.h, N, _ptr(q), _ptr(qd), _ptr(tau), _ptr(g), _ptr(fx), _ptr(out), _ptr(st),
                                threads, 1 if aba else 0))
        return out, st

    def fk(self, q, threads=0, scan=False):
        q = _F(q)
        N, n = q.shape[0], self.n
        out = np.empty((N, 12 * n), order="F")
        _chk(lib().orc_batch_fk(self.h, N, _ptr(q), _ptr(out), threads, 1 if scan else 0))
        return out.reshape(N, n, 12)

    def jacobian(self, q, frame, threads=0):
        q = _F(q)
        N, n = q.shape[0], self.n
        pose = np.empty((N, 12), order="F")
        J = np.empty((N, 6 * n), order="F")
        _chk(lib().orc_batch_jacobian(self.h, N, _ptr(q), frame.encode(), _ptr(pose), _ptr(J), threads))
        return pose, J.reshape(N, n, 6).transpose(0, 2, 1)

    def osc(self, q, qd, frame, target_R, target_p, kp, kd, accel_ff, posture, pkp, pkd, gravity=(0, 0, 9.81),
            eps=1e-6, threads=0):
        q, qd = _F(q), _F(qd)
        N, n = q.shape[0], self.n
        t12 = np.concatenate([np.asarray(target_R, dtype=np.float64).reshape(9), np.asarray(target_p, dtype=np.float64)])
        kp, kd, ff = (np.asarray(x, dtype=np.float64) for x in (kp, kd, accel_ff))
        post = np.asarray(posture, dtype=np.float64)
        g = np.asarray(gravity, dtype=np.float64)
        tau = np.empty((N, n), order="F")
        lam = np.empty((N, 36), order="F")
        st = np.zeros(N, dtype=np.int32)
        _chk(lib().orc_batch_osc(self.h, N, _ptr(q), _ptr(qd), frame.encode(), _ptr(t12), _ptr(kp), _ptr(kd),
                                 _ptr(ff), _ptr(post), pkp, pkd, _ptr(g), eps, _ptr(tau), _ptr(lam), _ptr(st), threads))
        return tau, lam.reshape(N, 6, 6).transpose(0, 2, 1), st

    def diff_ik(self, q, frame, target_R, target_p, kp, twist_ff, damping, threads=0):
        q = _F(q)
        N, n = q.shape[0], self.n
        t12 = np.concatenate([np.asarray(target_R, dtype=np.float64).reshape(9), np.asarray(target_p, dtype=np.float64)])
        kp, ff = (np.asarray(x, dtype=np.float64) for x in (kp, twist_ff))
        qdot = np.empty((N, n), order="F")
        err = np.empty((N, 6), order="F")
        _chk(lib().orc_batch_diffik(self.h, N, _ptr(q), frame.encode(), _ptr(t12), _ptr(kp), _ptr(ff), float(damping),
                                    _ptr(qdot), _ptr(err), threads))
        return qdot, err

    JVP_OPS = {"fk": (0, 12), "rnea": (1, 1), "crba": (2, None), "fd": (3, 1)}

    def jvp(self, op, x, dx, gravity=(0, 0, 9.81), fext=None, variant=0, threads=0):
        """(values, tangents[, status]) of op in {fk, rnea, crba, fd} run on duals.
        x / dx: tuples of (N, n) arrays (q[, qd, qdd|tau]); a None tangent is 0."""
        code, per = self.JVP_OPS[op]
        x = [_F(a) for a in x] + [None] * (3 - len(x))
        dx = [_F(a) for a in dx] + [None] * (3 - len(dx))
        N, n = x[0].shape[0], self.n
        K = n * n if per is None else n * per
        out = np.empty((N, K), order="F")
        dout = np.empty((N, K), order="F")
        st = np.zeros(N, dtype=np.int32)
        g = np.asarray(gravity, dtype=np.float64)
        fx = None if fext is None else np.asfortranarray(np.asarray(fext, dtype=np.float64).reshape(N, n * 6))
        _chk(lib().orc_batch_jvp(self.h, code, N, _ptr(x[0]), _ptr(x[1]), _ptr(x[2]), _ptr(dx[0]), _ptr(dx[1]),
                                 _ptr(dx[2]), _ptr(g), _ptr(fx), _ptr(out), _ptr(dout), _ptr(st), threads, variant))
        if op == "crba":
            out, dout = (a.reshape(N, n, n).transpose(0, 2, 1) for a in (out, dout))
        if op == "fd":
            return out, dout, st
        return out, dout

    def manipulability(self, q, frame, threads=0):
        q = _F(q)
        w = np.empty(q.shape[0])
        _chk(lib().orc_batch_manip(self.h, q.shape[0], _ptr(q), frame.encode(), _ptr(w), threads))
        return w

    def manipulability_jvp(self, q, dq, frame, threads=0):
        q, dq = _F(q), _F(dq)
        w, dw = np.empty(q.shape[0]), np.empty(q.shape[0])
        _chk(lib().orc_batch_manip_jvp(self.h, q.shape[0], _ptr(q), _ptr(dq), frame.encode(), _ptr(w), _ptr(dw),
                                       threads))
        return w, dw


def rel_err(a, b, axis=None):
    """proj/tests/helpers.hpp:67-72, per instance when axis is given: max|a-b| / max(1, max|a|, max|b|)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if axis is None:
        scale = max(1e-30, float(np.abs(a).max(initial=0)), float(np.abs(b).max(initial=0)))
        return float(np.abs(a - b).max(initial=0)) / max(1.0, scale)
    red = tuple(range(1, a.ndim))
    scale = np.maximum(np.maximum(np.abs(a).max(axis=red), np.abs(b).max(axis=red)), 1.0)
    return np.abs(a - b).max(axis=red) / scale

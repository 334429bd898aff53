"""B200-native batched rigid-body dynamics (the vecdyn hot path on sm_100a).

Python mirror of the reference C++ API (proj/core/include/vecdyn/*.hpp) over
the C-ABI in include/vecdyn_cuda.h.  Names, argument order and error types
follow the reference:

  robots.chain7() / humanoid23() / tree29() / by_name()      robots.cpp:12-32
  urdf.load_model(path) / load_model_from_string(text)       urdf.cpp:384-390
  RobotModel (dof, joints, frames, ancestor_mask, ...)        model.hpp:90-149
  floating_base(model)                                       model.cpp:289-331
  GravitySpec.standard() / zero() / from_field()              dynamics.hpp:35-50
  rnea, crba, gravity_vector, coriolis_vector,
  forward_dynamics (ABA), forward_kinematics,
  frame_transform, geometric_jacobian, osc_step               kinematics/dynamics/control.hpp
  StateBatch, random_states, batch_rnea, batch_crba,
  batch_forward_dynamics                                     batch.hpp:15-165

Batched device functions take CUDA torch tensors shaped (N, n) and return
(N, K) tensors; storage is the reference's column-major SoA (element (i, k)
at k*N + i), so results are views of (K, N) row-major buffers.  PyTorch is
used only for device memory and streams; all arithmetic runs in the
hand-written kernels of libvecdyn_cuda.so.
"""
import ctypes
import math

import numpy as np

from . import _lib
from ._lib import VD_F32, VD_F64

__all__ = [
    "Error", "DimensionError", "ModelError", "UnknownFrameError", "ParseError", "UnsupportedFeatureError",
    "UnsupportedStructureError", "SingularInertiaError", "CudaError", "RobotModel", "DeviceModel", "GravitySpec",
    "TaskGains", "TaskTarget", "PostureGains", "StateBatch", "robots", "urdf", "floating_base", "random_states",
    "rnea", "bias_forces", "gravity_vector", "coriolis_vector", "crba", "crba_packed", "unpack_crba", "forward_dynamics", "dynamics",
    "forward_kinematics", "forward_kinematics_scan", "frame_transform", "geometric_jacobian", "manipulability", "diff_ik_step", "osc_step", "batch_rnea", "batch_crba",
    "forward_kinematics_jvp", "rnea_jvp", "crba_jvp", "forward_dynamics_jvp", "rnea_derivatives",
    "forward_dynamics_derivatives", "manipulability_jvp", "jvp", "jvp_scalar", "jacobian_fwd", "lie_derivative",
    "batch_forward_dynamics", "batch_eval", "shard_range",
]


# ------------------------------------------------------------------ errors (errors.hpp:9-61)
class Error(RuntimeError):
    pass


class DimensionError(Error):
    pass


class ModelError(Error):
    pass


class UnknownFrameError(ModelError):
    pass


class ParseError(Error):
    def __init__(self, message, line=0, column=0):
        super().__init__(message)
        self.line = line
        self.column = column


class UnsupportedFeatureError(Error):
    pass


class UnsupportedStructureError(Error):
    pass


class SingularInertiaError(Error):
    pass


class CudaError(Error):
    pass


_CODES = {1: DimensionError, 2: ParseError, 3: ModelError, 4: UnknownFrameError, 5: UnsupportedFeatureError,
          6: UnsupportedStructureError, 7: SingularInertiaError, 8: CudaError, 9: ValueError, 10: Error, 11: Error}


def _check(rc):
    if rc == 0:
        return
    lib = _lib.load()
    msg = (lib.vd_last_error() or b"").decode()
    cls = _CODES.get(rc, Error)
    if cls is ParseError:
        raise ParseError(msg, lib.vd_last_error_line(), lib.vd_last_error_column())
    raise cls(msg)


def _buf(n):
    return ctypes.create_string_buffer(n)


# ------------------------------------------------------------------ model (host)
class RobotModel:
    """Immutable kinematic tree (model.hpp:90-149), owned by the C library."""

    def __init__(self, handle):
        self._h = ctypes.c_void_p(handle)
        self._lib = _lib.load()

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.vd_model_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def dof(self):
        return self._lib.vd_model_dof(self._h)

    @property
    def name(self):
        b = _buf(256)
        _check(self._lib.vd_model_name(self._h, b, 256))
        return b.value.decode()

    def max_depth(self):
        return self._lib.vd_model_max_depth(self._h)

    def is_serial_chain(self):
        return bool(self._lib.vd_model_is_serial_chain(self._h))

    def total_mass(self):
        return self._lib.vd_model_total_mass(self._h)

    def warnings(self):
        out = []
        for k in range(self._lib.vd_model_warning_count(self._h)):
            b = _buf(512)
            _check(self._lib.vd_model_warning(self._h, k, b, 512))
            out.append(b.value.decode())
        return out

    def parents(self):
        n = self.dof()
        arr = (ctypes.c_int * max(n, 1))()
        _check(self._lib.vd_model_parents(self._h, arr))
        return list(arr[:n])

    def joint_names(self):
        out = []
        for i in range(self.dof()):
            b = _buf(256)
            _check(self._lib.vd_model_joint_name(self._h, i, b, 256))
            out.append(b.value.decode())
        return out

    def joint_index(self, name):
        return self._lib.vd_model_joint_index(self._h, name.encode())

    def joint(self, i):
        """(type 0 revolute / 1 prismatic, axis[3], offset[12] R col-major + p, inertia 6x6)."""
        t = ctypes.c_int()
        ax = (ctypes.c_double * 3)()
        off = (ctypes.c_double * 12)()
        I = (ctypes.c_double * 36)()
        _check(self._lib.vd_model_joint(self._h, i, ctypes.byref(t), ax, off, I))
        return t.value, np.array(ax[:]), np.array(off[:]), np.array(I[:]).reshape(6, 6)

    def ancestor_mask(self):
        n = self.dof()
        m = (ctypes.c_double * max(n * n, 1))()
        _check(self._lib.vd_model_ancestor_mask(self._h, m))
        return np.array(m[: n * n]).reshape(n, n, order="F")

    def crba_pattern(self):
        """(rows, cols) of the branch-sparse lower triangle of M in
        compressed-column order (vd_model_crba_pattern); the layout of
        crba_packed's planes."""
        nnz = ctypes.c_int(0)
        _check(self._lib.vd_model_crba_pattern(self._h, None, None, ctypes.byref(nnz)))
        r = (ctypes.c_int32 * max(nnz.value, 1))()
        c = (ctypes.c_int32 * max(nnz.value, 1))()
        _check(self._lib.vd_model_crba_pattern(self._h, r, c, ctypes.byref(nnz)))
        return np.array(r[: nnz.value], dtype=np.int64), np.array(c[: nnz.value], dtype=np.int64)

    def frames(self):
        out = []
        for k in range(self._lib.vd_model_frame_count(self._h)):
            b = _buf(256)
            j = ctypes.c_int()
            off = (ctypes.c_double * 12)()
            _check(self._lib.vd_model_frame(self._h, k, b, 256, ctypes.byref(j), off))
            out.append((b.value.decode(), j.value, np.array(off[:])))
        return out

    def has_frame(self, name):
        return any(f[0] == name for f in self.frames())

    def frame_index(self, name):
        out = ctypes.c_int()
        _check(self._lib.vd_model_frame_index(self._h, name.encode(), ctypes.byref(out)))
        return out.value

    def fingerprint(self):
        return self._lib.vdi_model_fingerprint(self._h)


def _new_model(fn, *args):
    h = ctypes.c_void_p()
    _check(fn(*args, ctypes.byref(h)))
    return RobotModel(h.value)


class _Robots:
    """robots.hpp:11-20."""

    def by_name(self, name):
        return _new_model(_lib.load().vd_model_builtin, name.encode())

    def chain7(self):
        return self.by_name("chain7")

    def humanoid23(self):
        return self.by_name("humanoid23")

    def tree29(self):
        return self.by_name("tree29")

    def names(self):
        return ["chain7", "humanoid23", "tree29"]


class _Urdf:
    """urdf.hpp:66-71 (load entry points)."""

    def load_model(self, path):
        return _new_model(_lib.load().vd_model_load_urdf, path.encode())

    def load_model_from_string(self, text):
        data = text.encode() if isinstance(text, str) else text
        return _new_model(_lib.load().vd_model_load_urdf_string, data, len(data))


robots = _Robots()
urdf = _Urdf()


def floating_base(model):
    return _new_model(_lib.load().vd_model_floating_base, model.handle)


# ------------------------------------------------------------------ gravity / control structs
class GravitySpec:
    """a_g = −field; default (0, 0, +9.81) (dynamics.hpp:35-50)."""

    def __init__(self, linear_accel=(0.0, 0.0, 9.81)):
        self.accel = tuple(float(x) for x in linear_accel)

    @staticmethod
    def standard():
        return GravitySpec()

    @staticmethod
    def zero():
        return GravitySpec((0.0, 0.0, 0.0))

    @staticmethod
    def from_field(field):
        return GravitySpec(tuple(-float(x) for x in field))

    def c(self):
        return (ctypes.c_double * 3)(*self.accel)


class TaskGains:
    """control.hpp:12-22 (angular first)."""

    def __init__(self, kp=(0.0,) * 6, kd=(0.0,) * 6):
        self.kp = [float(x) for x in kp]
        self.kd = [float(x) for x in kd]

    @staticmethod
    def uniform(kp, kd=0.0):
        return TaskGains((kp,) * 6, (kd,) * 6)


class TaskTarget:
    """control.hpp:25-37; pose = (R 3x3, p 3)."""

    def __init__(self, frame, pose, gains=None, accel_ff=(0.0,) * 6, twist_ff=(0.0,) * 6):
        self.frame = frame
        self.pose = (np.asarray(pose[0], dtype=np.float64).reshape(3, 3), np.asarray(pose[1], dtype=np.float64))
        self.gains = gains or TaskGains()
        self.accel_ff = [float(x) for x in accel_ff]
        self.twist_ff = [float(x) for x in twist_ff]


class PostureGains:
    def __init__(self, kp=0.0, kd=0.0):
        self.kp = float(kp)
        self.kd = float(kd)


# ------------------------------------------------------------------ device model
class DeviceModel:
    """The model packed and uploaded to one GPU (compile-time specialised when it
    matches a builtin robot).  jit=True: for any other model, build (or reuse
    the cached) per-model module of generated routines and attach it to the
    model first (jit.py), with the task-space routines of `jit_frames`;
    ignored for the builtin robots."""

    def __init__(self, model, device=0, generic=False, jit=False, jit_frames=()):
        self.model = model
        self.device = int(device)
        self._lib = _lib.load()
        if jit and self._lib.vdi_model_fingerprint(model.handle) not in _builtin_fingerprints():
            from . import jit as _jit

            _jit.attach(model, frames=tuple(jit_frames))
        h = ctypes.c_void_p()
        _check(self._lib.vd_device_model_create(model.handle, self.device, ctypes.byref(h)))
        self._h = h
        if generic:
            _check(self._lib.vd_device_model_set_generic(self._h, 1))

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.vd_device_model_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def dof(self):
        return self._lib.vd_device_model_dof(self._h)

    def specialization(self):
        return self._lib.vd_device_model_specialization(self._h)

    def uses_jit(self):
        """True when calls run the model's JIT module (jit.py)."""
        return self._lib.vd_device_model_jit(self._h) == 1


_BUILTIN_FP = None


def _builtin_fingerprints():
    global _BUILTIN_FP
    if _BUILTIN_FP is None:
        _BUILTIN_FP = {_lib.load().vdi_model_fingerprint(robots.by_name(n).handle) for n in ("chain7", "tree29")}
    return _BUILTIN_FP


def _torch():
    import torch

    return torch


def _dtype_code(t):
    torch = _torch()
    if t.dtype == torch.float64:
        return VD_F64
    if t.dtype == torch.float32:
        return VD_F32
    raise TypeError("tensors must be float64 or float32")


def _soa(x, n, name, dtype=None, device=None):
    """(N, n) tensor -> (n, N) contiguous plane buffer on the model's device."""
    torch = _torch()
    if not torch.is_tensor(x):
        x = torch.as_tensor(np.asarray(x))
    if x.dim() == 1:
        x = x.unsqueeze(0)
    if x.dim() != 2 or x.shape[1] != n:
        raise DimensionError(f"{name} has shape {tuple(x.shape)}, model has {n} dof")
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    if device is not None and x.device != device:
        if x.is_cuda:
            # The C-ABI call runs under the model's device and stream; a tensor on
            # another GPU would be read with no ordering against its producer.
            raise CudaError(f"{name} is on {x.device}, the device model is on {device}")
        x = x.to(device)
    if not x.is_cuda:
        raise CudaError(f"{name} must be a CUDA tensor (no CPU fallback)")
    return _to_planes(x)


def _to_planes(x):
    """(N, K) CUDA tensor -> contiguous (K, N) planes.  Column-major input is
    already the plane layout (a view, no copy); row-major input goes through
    the library's staged transpose (vd_rows_to_planes), several times faster
    than a strided copy for these narrow shapes; anything else through torch."""
    torch = _torch()
    N, K = x.shape
    if N > 1 and K > 1 and x.stride() == (K, 1) and x.dtype in (torch.float64, torch.float32):
        out = torch.empty((K, N), dtype=x.dtype, device=x.device)
        with torch.cuda.device(x.device):  # the layout kernel runs on the current device
            _check(_lib.load().vd_rows_to_planes(_dtype_code(x), N, K, _p(x), K, _p(out), N, _stream(x.device)))
        return out
    return x.t().contiguous()


def _stream(dev):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _prep(dm, q, *others):
    torch = _torch()
    n = dm.dof()
    if not torch.is_tensor(q):
        q = torch.as_tensor(np.asarray(q))
    dev = torch.device("cuda", dm.device)
    qs = _soa(q, n, "q", device=dev)
    rest = [None if o is None else _soa(o, n, nm, dtype=qs.dtype, device=dev) for o, nm in others]
    return qs, rest, qs.shape[1], dev


def _out(dev, dtype, K, N):
    torch = _torch()
    return torch.empty((K, N), dtype=dtype, device=dev)


def _fext_planes(fext, N, n, dtype, dev):
    """fext: (N, n, 6) or (n, 6) world Plücker wrenches -> (6n, N) planes."""
    if fext is None:
        return None
    torch = _torch()
    if torch.is_tensor(fext) and fext.is_cuda and fext.device != dev:
        raise CudaError(f"external forces are on {fext.device}, the device model is on {dev}")
    f = torch.as_tensor(fext, dtype=dtype, device=dev)
    if f.dim() == 2:
        f = f.unsqueeze(0).expand(N, -1, -1)
    if tuple(f.shape) != (N, n, 6):
        raise DimensionError(f"external forces have shape {tuple(f.shape)}, expected ({N}, {n}, 6)")
    return _to_planes(f.reshape(N, 6 * n))


def _p(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _gravity(gravity, N, dtype, dev):
    """(gravity3 for the per-call entry point, None) for a GravitySpec or None;
    (None, (3, N) planes) for per-state gravity: an (N, 3) array of a_g = −field
    (vd_*_pg; the reference's GravitySpec is one per call, dynamics.hpp:35-50)."""
    if gravity is None or isinstance(gravity, GravitySpec):
        return (gravity or GravitySpec.standard()).c(), None
    torch = _torch()
    if torch.is_tensor(gravity) and gravity.is_cuda and gravity.device != dev:
        raise CudaError(f"gravity is on {gravity.device}, the device model is on {dev}")
    g = torch.as_tensor(gravity if torch.is_tensor(gravity) else np.asarray(gravity), dtype=dtype, device=dev)
    if tuple(g.shape) != (N, 3):
        raise DimensionError(f"per-state gravity has shape {tuple(g.shape)}, expected ({N}, 3)")
    if N == 0:
        return GravitySpec.standard().c(), None
    return None, _to_planes(g)


def rnea(dm, q, qd, qdd, gravity=None, fext=None):
    """rnea(model, q, qd, qdd, gravity, fext) — dynamics.hpp:250-267; (N, n) torques."""
    qs, (qds, qdds), N, dev = _prep(dm, q, (qd, "qd"), (qdd, "qdd"))
    n = dm.dof()
    out = _out(dev, qs.dtype, n, N)
    fx = _fext_planes(fext, N, n, qs.dtype, dev)
    g, gp = _gravity(gravity, N, qs.dtype, dev)
    lib = _lib.load()
    if gp is None:
        _check(lib.vd_rnea(dm.handle, _dtype_code(qs), N, _p(qs), _p(qds), _p(qdds), N, g, _p(fx), _p(out), N,
                           _stream(dev)))
    else:
        _check(lib.vd_rnea_pg(dm.handle, _dtype_code(qs), N, _p(qs), _p(qds), _p(qdds), N, _p(gp), _p(fx), _p(out), N,
                              _stream(dev)))
    return out.t()


def bias_forces(dm, q, qd, gravity=None, fext=None):
    """c + g (− Σ Jᵀ f_ext) = rnea(q, qd, 0) (dynamics.hpp:434-435)."""
    qs, (qds,), N, dev = _prep(dm, q, (qd, "qd"))
    n = dm.dof()
    out = _out(dev, qs.dtype, n, N)
    fx = _fext_planes(fext, N, n, qs.dtype, dev)
    g, gp = _gravity(gravity, N, qs.dtype, dev)
    lib = _lib.load()
    if gp is None:
        _check(lib.vd_bias(dm.handle, _dtype_code(qs), N, _p(qs), _p(qds), N, g, _p(fx), _p(out), N, _stream(dev)))
    else:
        _check(lib.vd_bias_pg(dm.handle, _dtype_code(qs), N, _p(qs), _p(qds), N, _p(gp), _p(fx), _p(out), N,
                              _stream(dev)))
    return out.t()


def gravity_vector(dm, q, gravity=None):
    """dynamics.hpp:402-408."""
    qs, _, N, dev = _prep(dm, q)
    out = _out(dev, qs.dtype, dm.dof(), N)
    g, gp = _gravity(gravity, N, qs.dtype, dev)
    lib = _lib.load()
    if gp is None:
        _check(lib.vd_gravity(dm.handle, _dtype_code(qs), N, _p(qs), N, g, _p(out), N, _stream(dev)))
    else:
        _check(lib.vd_gravity_pg(dm.handle, _dtype_code(qs), N, _p(qs), N, _p(gp), _p(out), N, _stream(dev)))
    return out.t()


def coriolis_vector(dm, q, qd):
    """dynamics.hpp:410-416."""
    qs, (qds,), N, dev = _prep(dm, q, (qd, "qd"))
    out = _out(dev, qs.dtype, dm.dof(), N)
    _check(_lib.load().vd_coriolis(dm.handle, _dtype_code(qs), N, _p(qs), _p(qds), N, _p(out), N, _stream(dev)))
    return out.t()


def crba(dm, q):
    """crba(model, q) — dynamics.hpp:352-365; returns (N, n, n)."""
    qs, _, N, dev = _prep(dm, q)
    n = dm.dof()
    out = _out(dev, qs.dtype, n * n, N)
    _check(_lib.load().vd_crba(dm.handle, _dtype_code(qs), N, _p(qs), N, _p(out), N, _stream(dev)))
    return out.t().reshape(N, n, n).transpose(1, 2)


def crba_packed(dm, q):
    """M(q) as its branch-sparse lower triangle: (N, nnz), column k =
    M[rows[k], cols[k]] for (rows, cols) = dm.model.crba_pattern().  Every
    other entry of the reference's dense M is an exact zero or the mirror of a
    packed one (dynamics.hpp:331-350); see unpack_crba."""
    qs, _, N, dev = _prep(dm, q)
    nnz = len(dm.model.crba_pattern()[0])
    out = _out(dev, qs.dtype, nnz, N)
    _check(_lib.load().vd_crba_packed(dm.handle, _dtype_code(qs), N, _p(qs), N, _p(out), N, _stream(dev)))
    return out.t()


def unpack_crba(model, Mp):
    """Dense symmetric (N, n, n) M from crba_packed's (N, nnz) output
    (symmetrize_lower, dynamics.hpp:331-335)."""
    torch = _torch()
    rows, cols = model.crba_pattern()
    n = model.dof()
    M = torch.zeros(Mp.shape[0], n, n, dtype=Mp.dtype, device=Mp.device)
    r = torch.as_tensor(rows, device=Mp.device)
    c = torch.as_tensor(cols, device=Mp.device)
    M[:, r, c] = Mp
    M[:, c, r] = Mp
    return M


def forward_dynamics(dm, q, qd, tau, gravity=None, fext=None, return_status=False):
    """forward_dynamics (dynamics.hpp:421-444) by the articulated-body algorithm.
    Raises SingularInertiaError when any instance is singular (the reference's
    LLT failure) unless return_status=True."""
    torch = _torch()
    qs, (qds, taus), N, dev = _prep(dm, q, (qd, "qd"), (tau, "tau"))
    n = dm.dof()
    out = _out(dev, qs.dtype, n, N)
    status = torch.zeros(N, dtype=torch.int32, device=dev)
    fx = _fext_planes(fext, N, n, qs.dtype, dev)
    g, gp = _gravity(gravity, N, qs.dtype, dev)
    lib = _lib.load()
    if gp is None:
        _check(lib.vd_aba(dm.handle, _dtype_code(qs), N, _p(qs), _p(qds), _p(taus), N, g, _p(fx), _p(out), N,
                          _p(status), _stream(dev)))
    else:
        _check(lib.vd_aba_pg(dm.handle, _dtype_code(qs), N, _p(qs), _p(qds), _p(taus), N, _p(gp), _p(fx), _p(out), N,
                             _p(status), _stream(dev)))
    if return_status:
        return out.t(), status
    if N and int(status.max().item()) != 0:
        raise SingularInertiaError(
            "forward_dynamics: mass matrix is not positive definite (zero-inertia degree of freedom?)")
    return out.t()


def dynamics(dm, q, qd, tau, gravity=None):
    """Fused M, bias and q̈ (BASELINE config 3); returns (M (N,n,n), bias (N,n), qdd (N,n), status)."""
    torch = _torch()
    qs, (qds, taus), N, dev = _prep(dm, q, (qd, "qd"), (tau, "tau"))
    n = dm.dof()
    M = _out(dev, qs.dtype, n * n, N)
    b = _out(dev, qs.dtype, n, N)
    a = _out(dev, qs.dtype, n, N)
    status = torch.zeros(N, dtype=torch.int32, device=dev)
    g, gp = _gravity(gravity, N, qs.dtype, dev)
    lib = _lib.load()
    if gp is None:
        _check(lib.vd_dynamics(dm.handle, _dtype_code(qs), N, _p(qs), _p(qds), _p(taus), N, g, _p(M), _p(b), _p(a), N,
                               _p(status), _stream(dev)))
    else:
        _check(lib.vd_dynamics_pg(dm.handle, _dtype_code(qs), N, _p(qs), _p(qds), _p(taus), N, _p(gp), _p(M), _p(b),
                                  _p(a), N, _p(status), _stream(dev)))
    return M.t().reshape(N, n, n).transpose(1, 2), b.t(), a.t(), status


def forward_kinematics(dm, q):
    """kinematics.hpp:43-56: (N, n, 12) with R column-major then p."""
    qs, _, N, dev = _prep(dm, q)
    n = dm.dof()
    out = _out(dev, qs.dtype, 12 * n, N)
    _check(_lib.load().vd_fk(dm.handle, _dtype_code(qs), N, _p(qs), N, _p(out), N, _stream(dev)))
    return out.t().reshape(N, n, 12)


def forward_kinematics_scan(dm, q):
    """kinematics.hpp:61-86 (serial chains; UnsupportedStructureError otherwise)."""
    qs, _, N, dev = _prep(dm, q)
    n = dm.dof()
    out = _out(dev, qs.dtype, 12 * n, N)
    _check(_lib.load().vd_fk_scan(dm.handle, _dtype_code(qs), N, _p(qs), N, _p(out), N, _stream(dev)))
    return out.t().reshape(N, n, 12)


def _frame_id(dm, frame):
    return frame if isinstance(frame, int) else dm.model.frame_index(frame)


def frame_transform(dm, q, frame):
    """kinematics.hpp:89-102: (N, 12) pose, R column-major then p."""
    qs, _, N, dev = _prep(dm, q)
    out = _out(dev, qs.dtype, 12, N)
    _check(_lib.load().vd_jacobian(dm.handle, _dtype_code(qs), N, _p(qs), N, _frame_id(dm, frame), _p(out), None, N,
                                   _stream(dev)))
    return out.t()


def geometric_jacobian(dm, q, frame):
    """kinematics.hpp:108-136: (N, 6, n)."""
    qs, _, N, dev = _prep(dm, q)
    n = dm.dof()
    out = _out(dev, qs.dtype, 6 * n, N)
    _check(_lib.load().vd_jacobian(dm.handle, _dtype_code(qs), N, _p(qs), N, _frame_id(dm, frame), None, _p(out), N,
                                   _stream(dev)))
    return out.t().reshape(N, n, 6).transpose(1, 2)


# ------------------------------------------------------------------ forward-mode JVPs (autodiff.hpp:41-56)
# jvp(fn, x, v) of the reference, for fn in the library's own batched
# functions: one device pass on dual numbers returns (fn(x), D fn(x)·v).
# Tangent arguments default to zero.
def forward_kinematics_jvp(dm, q, dq):
    """(frames, d frames), both (N, n, 12) like forward_kinematics."""
    qs, (dqs,), N, dev = _prep(dm, q, (dq, "dq"))
    n = dm.dof()
    out, dout = _out(dev, qs.dtype, 12 * n, N), _out(dev, qs.dtype, 12 * n, N)
    _check(_lib.load().vd_fk_jvp(dm.handle, _dtype_code(qs), N, _p(qs), _p(dqs), N, _p(out), _p(dout), N,
                                 _stream(dev)))
    return out.t().reshape(N, n, 12), dout.t().reshape(N, n, 12)


def rnea_jvp(dm, q, qd, qdd, dq=None, dqd=None, dqdd=None, gravity=None, fext=None):
    """(τ, dτ) with dτ = ∂τ/∂q·dq + ∂τ/∂q̇·dq̇ + ∂τ/∂q̈·dq̈ (fext held constant)."""
    qs, (qds, qdds, dqs, dqds, dqdds), N, dev = _prep(dm, q, (qd, "qd"), (qdd, "qdd"), (dq, "dq"), (dqd, "dqd"),
                                                        (dqdd, "dqdd"))
    n = dm.dof()
    out, dout = _out(dev, qs.dtype, n, N), _out(dev, qs.dtype, n, N)
    fx = _fext_planes(fext, N, n, qs.dtype, dev)
    g = (gravity or GravitySpec.standard()).c()
    _check(_lib.load().vd_rnea_jvp(dm.handle, _dtype_code(qs), N, _p(qs), _p(qds), _p(qdds), _p(dqs), _p(dqds),
                                   _p(dqdds), N, g, _p(fx), _p(out), _p(dout), N, _stream(dev)))
    return out.t(), dout.t()


def crba_jvp(dm, q, dq):
    """(M, dM) with dM = Σ_k ∂M/∂q_k dq_k, both (N, n, n)."""
    qs, (dqs,), N, dev = _prep(dm, q, (dq, "dq"))
    n = dm.dof()
    out, dout = _out(dev, qs.dtype, n * n, N), _out(dev, qs.dtype, n * n, N)
    _check(_lib.load().vd_crba_jvp(dm.handle, _dtype_code(qs), N, _p(qs), _p(dqs), N, _p(out), _p(dout), N,
                                   _stream(dev)))
    return (out.t().reshape(N, n, n).transpose(1, 2), dout.t().reshape(N, n, n).transpose(1, 2))


def forward_dynamics_jvp(dm, q, qd, tau, dq=None, dqd=None, dtau=None, gravity=None, fext=None,
                         return_status=False):
    """(q̈, dq̈) by the articulated-body algorithm on duals (the G1 builtin:
    dq̈ = M⁻¹(dτ − ∂ID·(dq, dq̇)) from its ABA and RNEA-JVP, q̈ bit for bit the
    plain forward_dynamics); SingularInertiaError as forward_dynamics unless
    return_status."""
    torch = _torch()
    qs, (qds, taus, dqs, dqds, dtaus), N, dev = _prep(dm, q, (qd, "qd"), (tau, "tau"), (dq, "dq"), (dqd, "dqd"),
                                                        (dtau, "dtau"))
    n = dm.dof()
    out, dout = _out(dev, qs.dtype, n, N), _out(dev, qs.dtype, n, N)
    status = torch.zeros(N, dtype=torch.int32, device=dev)
    fx = _fext_planes(fext, N, n, qs.dtype, dev)
    g = (gravity or GravitySpec.standard()).c()
    _check(_lib.load().vd_aba_jvp(dm.handle, _dtype_code(qs), N, _p(qs), _p(qds), _p(taus), _p(dqs), _p(dqds),
                                  _p(dtaus), N, g, _p(fx), _p(out), _p(dout), N, _p(status), _stream(dev)))
    if return_status:
        return out.t(), dout.t(), status
    if N and int(status.max().item()) != 0:
        raise SingularInertiaError(
            "forward_dynamics: mass matrix is not positive definite (zero-inertia degree of freedom?)")
    return out.t(), dout.t()


def rnea_derivatives(dm, q, qd, qdd, gravity=None):
    """(∂τ/∂q, ∂τ/∂q̇), each (N, n, n) with column j = the JVP along e_j:
    jacobian_fwd (autodiff.hpp:67-84) of the batched RNEA, n passes of the
    dual-number kernel per argument (∂τ/∂q̈ is M, crba)."""
    return _jac_fwd(dm, q, lambda e, zero: rnea_jvp(dm, q, qd, qdd, e, zero, zero, gravity)[1],
                    lambda e, zero: rnea_jvp(dm, q, qd, qdd, zero, e, zero, gravity)[1])


def forward_dynamics_derivatives(dm, q, qd, tau, gravity=None):
    """(∂q̈/∂q, ∂q̈/∂q̇, ∂q̈/∂τ), each (N, n, n): jacobian_fwd (autodiff.hpp:67-84)
    of forward dynamics by the library's ABA-JVP (the dual-number ABA; for the
    G1 its implicit-function form), n passes per argument (∂q̈/∂τ = M⁻¹).
    SingularInertiaError as forward_dynamics."""
    return _jac_fwd(dm, q, lambda e, zero: forward_dynamics_jvp(dm, q, qd, tau, e, zero, zero, gravity)[1],
                    lambda e, zero: forward_dynamics_jvp(dm, q, qd, tau, zero, e, zero, gravity)[1],
                    lambda e, zero: forward_dynamics_jvp(dm, q, qd, tau, zero, zero, e, gravity)[1])


def _jac_fwd(dm, q, *tangent_fns):
    torch = _torch()
    qs = q if torch.is_tensor(q) else torch.as_tensor(np.asarray(q))
    N, n = qs.shape[0], dm.dof()
    dev = torch.device("cuda", dm.device)
    dtype = qs.dtype if qs.dtype in (torch.float64, torch.float32) else torch.float64
    zero = torch.zeros((N, n), dtype=dtype, device=dev)
    outs = []
    for fn in tangent_fns:
        J = torch.empty((N, n, n), dtype=dtype, device=dev)
        for j in range(n):
            e = torch.zeros((N, n), dtype=dtype, device=dev)
            e[:, j] = 1
            J[:, :, j] = fn(e, zero)
        outs.append(J)
    return tuple(outs)


def manipulability(dm, q, frame):
    """manipulability(geometric_jacobian(frame)) (kinematics.hpp:138-153): (N,),
    0 at singular configurations."""
    qs, _, N, dev = _prep(dm, q)
    out = _out(dev, qs.dtype, 1, N)
    _check(_lib.load().vd_manipulability(dm.handle, _dtype_code(qs), N, _p(qs), N, _frame_id(dm, frame), _p(out),
                                         _stream(dev)))
    return out.reshape(N)


def manipulability_jvp(dm, q, dq, frame):
    """(w, D w(q)·dq), each (N,): jvp_scalar (autodiff.hpp:52-62) of
    manipulability(geometric_jacobian(frame)) (kinematics.hpp:138-153) on
    dual numbers; the tangent is 0 where the Gram matrix does not factor."""
    qs, (dqs,), N, dev = _prep(dm, q, (dq, "dq"))
    w = _out(dev, qs.dtype, 1, N)
    dw = _out(dev, qs.dtype, 1, N)
    _check(_lib.load().vd_manipulability_jvp(dm.handle, _dtype_code(qs), N, _p(qs), _p(dqs), N, _frame_id(dm, frame),
                                             _p(w), _p(dw), _stream(dev)))
    return w.reshape(N), dw.reshape(N)


def jvp(h, x, v):
    """jvp (autodiff.hpp:41-50), batched: (h(x), Dh(x)·v) from a JVP function
    h(x, dx) -> (value, tangent) over N states (the library's *_jvp entry
    points, e.g. ``lambda q, dq: forward_kinematics_jvp(dm, q, dq)``).
    DimensionError when v's shape is not x's (autodiff.hpp:44-48)."""
    if tuple(v.shape) != tuple(x.shape):
        raise DimensionError(f"jvp: tangent has shape {tuple(v.shape)}, input has {tuple(x.shape)}")
    return h(x, v)


def jvp_scalar(h, x, v):
    """jvp_scalar (autodiff.hpp:52-62), batched: h returns (N,) values and tangents."""
    val, tan = jvp(h, x, v)
    if val.dim() != 1 or tan.dim() != 1:
        raise DimensionError("jvp_scalar: the function is not scalar-valued per state")
    return val, tan


def jacobian_fwd(h, x):
    """jacobian_fwd (autodiff.hpp:64-84), batched: the (N, m, d) Jacobian of h
    at the N states x (N, d), column j from one JVP pass along e_j (an AD
    Jacobian costs d passes; the reference says the same)."""
    torch = _torch()
    N, d = x.shape
    cols = []
    for j in range(d):
        e = torch.zeros_like(x)
        e[:, j] = 1
        t = h(x, e)[1]
        cols.append(t.reshape(N, -1))
    if not cols:
        return torch.empty((N, 0, 0), dtype=x.dtype, device=x.device)
    return torch.stack(cols, dim=2)


def lie_derivative(h, f, z):
    """L_f h(z) = ⟨∇h(z), f(z)⟩ as one JVP of h along f(z), the gradient never
    formed (control.hpp:157-163), batched: z is a tensor of N states (any
    trailing shape), f(z) a vector field of z's shape and h(z, dz) -> (value,
    tangent) a JVP of the scalar function, e.g. ``lambda z, dz:
    manipulability_jvp(dm, z[:, :n], dz[:, :n], frame)``.  Returns the (N,)
    tangents."""
    direction = f(z)
    if tuple(direction.shape) != tuple(z.shape):
        raise DimensionError(f"lie_derivative: f(z) has shape {tuple(direction.shape)}, z has {tuple(z.shape)}")
    return h(z, direction)[1]


def diff_ik_step(dm, q, target, damping, return_error=False):
    """diff_ik_step (control.hpp:79-97) for a batch sharing one target: (N, n) q̇;
    with return_error also the (N, 6) pose error."""
    qs, _, N, dev = _prep(dm, q)
    n = dm.dof()
    P = _lib.TaskParams()
    P.frame = _frame_id(dm, target.frame)
    R, p = target.pose
    for c in range(3):
        for r in range(3):
            P.target[c * 3 + r] = float(R[r][c])
    for k in range(3):
        P.target[9 + k] = float(p[k])
    for k in range(6):
        P.kp[k] = target.gains.kp[k]
        P.twist_ff[k] = target.twist_ff[k]
    P.damping = float(damping)
    qdot = _out(dev, qs.dtype, n, N)
    err = _out(dev, qs.dtype, 6, N) if return_error else None
    _check(_lib.load().vd_diff_ik(dm.handle, _dtype_code(qs), N, _p(qs), N, ctypes.byref(P), _p(qdot), _p(err), N,
                                  None, _stream(dev)))
    return (qdot.t(), err.t()) if return_error else qdot.t()


def osc_step(dm, q, qd, target, posture, posture_gains, gravity=None, epsilon=1e-6, return_lambda=False,
             return_status=False):
    """osc_step (control.hpp:108-155) for a batch sharing one target/posture."""
    torch = _torch()
    qs, (qds,), N, dev = _prep(dm, q, (qd, "qd"))
    n = dm.dof()
    P = _lib.OscParams()
    P.frame = _frame_id(dm, target.frame)
    R, p = target.pose
    for c in range(3):
        for r in range(3):
            P.target[c * 3 + r] = float(R[r][c])
    for k in range(3):
        P.target[9 + k] = float(p[k])
    for k in range(6):
        P.kp[k] = target.gains.kp[k]
        P.kd[k] = target.gains.kd[k]
        P.accel_ff[k] = target.accel_ff[k]
    post = (ctypes.c_double * max(n, 1))(*[float(x) for x in np.asarray(posture, dtype=np.float64).reshape(-1)])
    P.posture = ctypes.cast(post, _lib.Pd)
    P.posture_kp = posture_gains.kp
    P.posture_kd = posture_gains.kd
    g = (gravity or GravitySpec.standard()).accel
    for k in range(3):
        P.gravity[k] = g[k]
    P.epsilon = float(epsilon)
    tau = _out(dev, qs.dtype, n, N)
    lam = _out(dev, qs.dtype, 36, N) if return_lambda else None
    status = torch.zeros(N, dtype=torch.int32, device=dev)
    _check(_lib.load().vd_osc(dm.handle, _dtype_code(qs), N, _p(qs), _p(qds), N, ctypes.byref(P), _p(tau), _p(lam), N,
                              _p(status), _stream(dev)))
    if not return_status and N and int(status.max().item()) != 0:
        raise SingularInertiaError("osc_step: mass matrix is not positive definite")
    out = [tau.t()]
    if return_lambda:
        out.append(lam.t().reshape(N, 6, 6).transpose(1, 2))
    if return_status:
        out.append(status)
    return out[0] if len(out) == 1 else tuple(out)


# ------------------------------------------------------------------ batch layer (batch.hpp)
class StateBatch:
    """batch.hpp:15-45; arrays are (N, n) float64, column-major (Fortran) order."""

    def __init__(self, q, qd, qdd=None, tau=None):
        self.q, self.qd, self.qdd, self.tau = q, qd, qdd, tau

    def size(self):
        return int(self.q.shape[0])

    def validate(self, model):
        n = model.dof()
        if self.q.shape[1] != n:
            raise DimensionError(f"StateBatch: q has {self.q.shape[1]} columns, model has {n} dof")
        for name in ("qd", "qdd", "tau"):
            m = getattr(self, name)
            if m is not None and m.size and m.shape != self.q.shape:
                raise DimensionError(f"StateBatch: {name} is {m.shape[0]}x{m.shape[1]}, expected "
                                     f"{self.q.shape[0]}x{n}")


def random_states(model, count, seed, with_qdd=True, with_tau=False):
    """batch.hpp:48-75 — bit-identical mt19937_64 stream."""
    n = model.dof()
    arrs = [np.empty((count, n), dtype=np.float64, order="F") for _ in range(4)]
    q, qd, qdd, tau = arrs
    ptr = lambda a, on: ctypes.c_void_p(a.ctypes.data if on else 0)  # noqa: E731
    _check(_lib.load().vd_random_states(model.handle, count, seed, ptr(q, True), ptr(qd, True), ptr(qdd, with_qdd),
                                        ptr(tau, with_tau)))
    return StateBatch(q, qd, qdd if with_qdd else None, tau if with_tau else None)


def _host_f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _devices(devices):
    if devices is None:
        devices = [0]
    arr = (ctypes.c_int * len(devices))(*devices)
    return arr, len(devices)


def batch_rnea(model, batch, gravity=None, devices=None):
    """batch.hpp:128-138 with a device list instead of `workers`."""
    batch.validate(model)
    N, n = batch.size(), model.dof()
    out = np.empty((N, n), dtype=np.float64, order="F")
    q, qd, qdd = _host_f(batch.q), _host_f(batch.qd), _host_f(batch.qdd)
    d, nd = _devices(devices)
    g = (gravity or GravitySpec.standard()).c()
    _check(_lib.load().vd_batch_rnea_host(model.handle, N, q.ctypes.data, qd.ctypes.data, qdd.ctypes.data, g,
                                          out.ctypes.data, d, nd))
    return out


def batch_crba(model, batch, devices=None):
    """batch.hpp:141-151: rows are column-major flattened n x n matrices."""
    batch.validate(model)
    N, n = batch.size(), model.dof()
    out = np.empty((N, n * n), dtype=np.float64, order="F")
    q = _host_f(batch.q)
    d, nd = _devices(devices)
    _check(_lib.load().vd_batch_crba_host(model.handle, N, q.ctypes.data, out.ctypes.data, d, nd))
    return out


def batch_forward_dynamics(model, batch, gravity=None, devices=None):
    """batch.hpp:154-165 (ABA on the device)."""
    batch.validate(model)
    N, n = batch.size(), model.dof()
    out = np.empty((N, n), dtype=np.float64, order="F")
    q, qd, tau = _host_f(batch.q), _host_f(batch.qd), _host_f(batch.tau)
    d, nd = _devices(devices)
    g = (gravity or GravitySpec.standard()).c()
    _check(_lib.load().vd_batch_forward_dynamics_host(model.handle, N, q.ctypes.data, qd.ctypes.data, tau.ctypes.data,
                                                      g, out.ctypes.data, None, d, nd))
    return out


class _ShardStates:
    """One device's shard of a StateBatch for batch_eval: (N_shard, n) views
    of plane buffers on the device (None for an absent field), the layout
    every entry point reads without a copy."""

    def __init__(self, batch, b, e, dev):
        torch = _torch()

        def up(a):
            if a is None or not a.size:
                return None
            return torch.from_numpy(np.ascontiguousarray(a[b:e].T)).to(dev, non_blocking=False).t()

        self.q, self.qd, self.qdd, self.tau = (up(a) for a in (batch.q, batch.qd, batch.qdd, batch.tau))
        self.begin, self.end = b, e


def batch_eval(model, batch, fn, devices=None):
    """batch_eval (batch.hpp:76-126) with a device list instead of `workers`:
    the batch is cut into contiguous shards (shard_range, the reference's
    chunk rule) and fn(device_model, states) runs once per shard on its
    device, one host thread per device; `states` holds the shard's q, qd,
    qdd, tau as (N_shard, n) CUDA tensors, and fn returns an (N_shard, K)
    tensor (or array).  fn sees whole shards rather than single states (the
    library's entry points are batched); every state still runs the same code
    path whatever the partition, so the (N, K) result is bitwise identical
    for any device list.  N = 0 gives a 0 x 0 array, as the reference."""
    import threading

    torch = _torch()
    batch.validate(model)
    N = batch.size()
    if N == 0:
        return np.empty((0, 0), dtype=np.float64, order="F")
    devices = list(devices) if devices else [0]
    world = min(len(devices), N)
    parts, errors = [None] * world, [None] * world

    def work(k):
        try:
            b, e = shard_range(N, world, k)
            dev = torch.device("cuda", devices[k])
            with torch.cuda.device(dev):
                dm = DeviceModel(model, devices[k])
                y = fn(dm, _ShardStates(batch, b, e, dev))
                y = y.detach().double().cpu().numpy() if torch.is_tensor(y) else np.asarray(y, dtype=np.float64)
            if y.ndim == 1:
                y = y[:, None]
            if y.shape[0] != e - b:
                raise DimensionError(f"batch_eval: fn returned {y.shape[0]} rows for a shard of {e - b} states")
            parts[k] = y
        except BaseException as exc:  # re-raised on the calling thread
            errors[k] = exc

    threads = [threading.Thread(target=work, args=(k,)) for k in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for exc in errors:
        if exc is not None:
            raise exc
    if len({p.shape[1] for p in parts}) != 1:
        raise DimensionError("batch_eval: fn returned different widths on different shards")
    return np.asfortranarray(np.concatenate(parts, axis=0))


def shard_range(N, world, rank):
    """Contiguous shard of N instances for `rank` of `world` (batch.hpp:111-119 rule)."""
    b, e = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.load().vd_shard_range(N, world, rank, ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


# Fail loudly at import time when the native library is absent.
_lib.load()
_ = math

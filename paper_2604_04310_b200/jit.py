"""Per-model JIT modules: the generated straight-line routines for a model
that is not one of the compile-time robots (chain7, tree29).

The library ships generated kernels only for its builtin robots; any other
URDF runs the loop ("runtime view") kernels, which keep per-joint state in
local memory and are 5-10x slower.  `build(model)` runs the same generator
(codegen.py) on the model's packed tree, compiles the routines with nvcc for
sm_100a into a shared library (csrc/vd_jit_entry.cuh's entry points) and
caches it by model fingerprint and source hash; `attach(model)` loads it into
the model (vd_model_attach_jit) so every device model created from it
afterwards runs ABA, RNEA, bias, gravity, Coriolis, CRBA, packed CRBA and FK
through it, and OSC / Jacobian / diff-IK / manipulability on the frames the
module was built for.  JVPs stay on the loop kernels.

    python -m paper_2604_04310_b200.jit robot.urdf [frame ...]   # prints the module path

C++ users attach the printed module with vd_model_attach_jit.
"""
import hashlib
import os
import subprocess
import sys
import tempfile

from . import _lib
from . import codegen

_HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(_HERE, "csrc")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++20",
              "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared"]


def cache_dir():
    """VD_JIT_CACHE, else paper_2604_04310_b200/lib/jit (in-tree, git-ignored)."""
    return os.environ.get("VD_JIT_CACHE") or os.path.join(_HERE, "lib", "jit")


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def frame_joints(model, frames):
    """Joint indices of named frames (vd_model_frame); UnknownFrameError-like
    RuntimeError for a name the model does not have."""
    import ctypes

    lib = _lib.load()
    out = []
    for name in frames:
        k = ctypes.c_int()
        if lib.vd_model_frame_index(model.handle, name.encode(), ctypes.byref(k)) != 0:
            raise RuntimeError(lib.vd_last_error().decode())
        j = ctypes.c_int()
        buf = ctypes.create_string_buffer(256)
        off = (ctypes.c_double * 12)()
        lib.vd_model_frame(model.handle, k.value, buf, 256, ctypes.byref(j), off)
        if j.value >= 0:
            out.append(j.value)
    return sorted(set(out))


def source(model, frames=()):
    """(translation unit text, model fingerprint) for `model` (a RobotModel);
    `frames`: frame names whose OSC / Jacobian / diff-IK / manipulability
    routines the module also carries."""
    return codegen.jit_source(_lib.load(), model.handle, task_joints=frame_joints(model, frames))


def build(model, frames=(), verbose=False):
    """Path of the model's JIT module, compiling it if it is not cached.
    Raises RuntimeError with nvcc's output if the compile fails."""
    src, fp = source(model, frames)
    # the cache key covers everything the module is compiled from: its source,
    # the flags and the library headers it includes (launch machinery, kernel
    # templates, the Launch struct of the library it will be loaded into)
    h = hashlib.sha1((src + " ".join(NVCC_FLAGS)).encode())
    for name in sorted(os.listdir(CSRC)):
        if name.endswith((".cuh", ".hpp", ".h")) and name != "vd_gen_robots.cuh":
            with open(os.path.join(CSRC, name), "rb") as f:
                h.update(f.read())
    tag = h.hexdigest()[:12]
    out_dir = cache_dir()
    os.makedirs(out_dir, exist_ok=True)
    so = os.path.join(out_dir, f"vdj_{fp:016x}_{tag}.so")
    if os.path.exists(so):
        return so
    with tempfile.TemporaryDirectory(dir=out_dir) as tmp:
        cu = os.path.join(tmp, "jit.cu")
        with open(cu, "w") as f:
            f.write(src)
        tmp_so = os.path.join(tmp, "jit.so")
        cmd = [_nvcc()] + NVCC_FLAGS + ["-I", CSRC, cu, "-o", tmp_so]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"JIT compile failed ({' '.join(cmd)}):\n{r.stdout}{r.stderr}")
        os.replace(tmp_so, so)  # atomic: concurrent builders of the same model agree
    return so


def attach(model, path=None, frames=(), verbose=False):
    """Attach a JIT module (built if `path` is None, with the task-space
    routines of `frames`) to `model`; device models created from it
    afterwards use it.  Returns the module path (None for a model without
    joints: every call on it is a no-op already)."""
    if model.dof() == 0:
        return None
    path = path or build(model, frames=frames, verbose=verbose)
    lib = _lib.load()
    if lib.vd_model_attach_jit(model.handle, path.encode()) != 0:
        raise RuntimeError(lib.vd_last_error().decode())
    return path


def main(argv):
    from . import urdf

    if not argv:
        sys.stderr.write("usage: python -m paper_2604_04310_b200.jit robot.urdf [frame ...]\n")
        return 2
    print(build(urdf.load_model(argv[0]), frames=argv[1:], verbose=True))
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))

"""ctypes binding of the C-ABI in include/vecdyn_cuda.h.

The shared library is built in-tree (paper_2604_04310_b200/lib/) by
__graft_entry__.build().  There is no fallback: if the library is missing the
import fails loudly.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VD_LIB_PATH") or os.path.join(_HERE, "lib", "libvecdyn_cuda.so")

VD_OK = 0
VD_ERR_DIMENSION = 1
VD_ERR_PARSE = 2
VD_ERR_MODEL = 3
VD_ERR_UNKNOWN_FRAME = 4
VD_ERR_UNSUPPORTED_FEATURE = 5
VD_ERR_UNSUPPORTED_STRUCTURE = 6
VD_ERR_SINGULAR_INERTIA = 7
VD_ERR_CUDA = 8
VD_ERR_INVALID_ARGUMENT = 9
VD_ERR_IO = 10
VD_ERR_GENERIC = 11
VD_F64 = 0
VD_F32 = 1

c_int, c_int64, c_double, c_void_p, c_char_p, c_size_t, c_uint64 = (
    ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t, ctypes.c_uint64)
P = c_void_p
Pi = ctypes.POINTER(c_int)
Pd = ctypes.POINTER(c_double)


class OscParams(ctypes.Structure):
    _fields_ = [("frame", c_int), ("target", c_double * 12), ("kp", c_double * 6), ("kd", c_double * 6),
                ("accel_ff", c_double * 6), ("posture", Pd), ("posture_kp", c_double), ("posture_kd", c_double),
                ("gravity", c_double * 3), ("epsilon", c_double)]


class TaskParams(ctypes.Structure):
    _fields_ = [("frame", c_int), ("target", c_double * 12), ("kp", c_double * 6), ("twist_ff", c_double * 6),
                ("damping", c_double)]


# name -> (restype, argtypes); mirrors include/vecdyn_cuda.h one for one.
SIGNATURES = {
    "vd_last_error": (c_char_p, []),
    "vd_last_error_line": (c_int, []),
    "vd_last_error_column": (c_int, []),
    "vd_version": (c_char_p, []),
    "vd_model_builtin": (c_int, [c_char_p, ctypes.POINTER(c_void_p)]),
    "vd_model_load_urdf": (c_int, [c_char_p, ctypes.POINTER(c_void_p)]),
    "vd_model_load_urdf_string": (c_int, [c_char_p, c_size_t, ctypes.POINTER(c_void_p)]),
    "vd_model_floating_base": (c_int, [P, ctypes.POINTER(c_void_p)]),
    "vd_model_destroy": (None, [P]),
    "vd_model_dof": (c_int, [P]),
    "vd_model_max_depth": (c_int, [P]),
    "vd_model_is_serial_chain": (c_int, [P]),
    "vd_model_total_mass": (c_double, [P]),
    "vd_model_warning_count": (c_int, [P]),
    "vd_model_warning": (c_int, [P, c_int, ctypes.c_char_p, c_size_t]),
    "vd_model_name": (c_int, [P, ctypes.c_char_p, c_size_t]),
    "vd_model_parents": (c_int, [P, Pi]),
    "vd_model_joint_name": (c_int, [P, c_int, ctypes.c_char_p, c_size_t]),
    "vd_model_joint_index": (c_int, [P, c_char_p]),
    "vd_model_joint": (c_int, [P, c_int, Pi, Pd, Pd, Pd]),
    "vd_model_ancestor_mask": (c_int, [P, Pd]),
    "vd_model_crba_pattern": (c_int, [P, P, P, P]),
    "vd_model_frame_count": (c_int, [P]),
    "vd_model_frame": (c_int, [P, c_int, ctypes.c_char_p, c_size_t, Pi, Pd]),
    "vd_model_frame_index": (c_int, [P, c_char_p, Pi]),
    "vd_random_states": (c_int, [P, c_int64, c_uint64, P, P, P, P]),
    "vd_device_model_create": (c_int, [P, c_int, ctypes.POINTER(c_void_p)]),
    "vd_device_model_destroy": (None, [P]),
    "vd_device_model_dof": (c_int, [P]),
    "vd_device_model_specialization": (c_int, [P]),
    "vd_device_model_set_generic": (c_int, [P, c_int]),
    "vd_model_attach_jit": (c_int, [P, c_char_p]),
    "vd_device_model_jit": (c_int, [P]),
    "vd_fk": (c_int, [P, c_int, c_int64, P, c_int64, P, c_int64, P]),
    "vd_fk_scan": (c_int, [P, c_int, c_int64, P, c_int64, P, c_int64, P]),
    "vd_jacobian": (c_int, [P, c_int, c_int64, P, c_int64, c_int, P, P, c_int64, P]),
    "vd_rnea": (c_int, [P, c_int, c_int64, P, P, P, c_int64, Pd, P, P, c_int64, P]),
    "vd_bias": (c_int, [P, c_int, c_int64, P, P, c_int64, Pd, P, P, c_int64, P]),
    "vd_gravity": (c_int, [P, c_int, c_int64, P, c_int64, Pd, P, c_int64, P]),
    "vd_coriolis": (c_int, [P, c_int, c_int64, P, P, c_int64, P, c_int64, P]),
    "vd_crba": (c_int, [P, c_int, c_int64, P, c_int64, P, c_int64, P]),
    "vd_crba_packed": (c_int, [P, c_int, c_int64, P, c_int64, P, c_int64, P]),
    "vd_aba": (c_int, [P, c_int, c_int64, P, P, P, c_int64, Pd, P, P, c_int64, P, P]),
    "vd_dynamics": (c_int, [P, c_int, c_int64, P, P, P, c_int64, Pd, P, P, P, c_int64, P, P]),
    "vd_rnea_pg": (c_int, [P, c_int, c_int64, P, P, P, c_int64, P, P, P, c_int64, P]),
    "vd_bias_pg": (c_int, [P, c_int, c_int64, P, P, c_int64, P, P, P, c_int64, P]),
    "vd_gravity_pg": (c_int, [P, c_int, c_int64, P, c_int64, P, P, c_int64, P]),
    "vd_aba_pg": (c_int, [P, c_int, c_int64, P, P, P, c_int64, P, P, P, c_int64, P, P]),
    "vd_dynamics_pg": (c_int, [P, c_int, c_int64, P, P, P, c_int64, P, P, P, P, c_int64, P, P]),
    "vd_osc": (c_int, [P, c_int, c_int64, P, P, c_int64, ctypes.POINTER(OscParams), P, P, c_int64, P, P]),
    "vd_diff_ik": (c_int, [P, c_int, c_int64, P, c_int64, ctypes.POINTER(TaskParams), P, P, c_int64, P, P]),
    "vd_manipulability": (c_int, [P, c_int, c_int64, P, c_int64, c_int, P, P]),
    "vd_manipulability_jvp": (c_int, [P, c_int, c_int64, P, P, c_int64, c_int, P, P, P]),
    "vd_fk_jvp": (c_int, [P, c_int, c_int64, P, P, c_int64, P, P, c_int64, P]),
    "vd_rnea_jvp": (c_int, [P, c_int, c_int64, P, P, P, P, P, P, c_int64, Pd, P, P, P, c_int64, P]),
    "vd_crba_jvp": (c_int, [P, c_int, c_int64, P, P, c_int64, P, P, c_int64, P]),
    "vd_aba_jvp": (c_int, [P, c_int, c_int64, P, P, P, P, P, P, c_int64, Pd, P, P, P, c_int64, P, P]),
    "vd_batch_rnea_host": (c_int, [P, c_int64, P, P, P, Pd, P, Pi, c_int]),
    "vd_batch_crba_host": (c_int, [P, c_int64, P, P, Pi, c_int]),
    "vd_batch_forward_dynamics_host": (c_int, [P, c_int64, P, P, P, Pd, P, P, Pi, c_int]),
    "vd_shard_range": (c_int, [c_int64, c_int, c_int, ctypes.POINTER(c_int64), ctypes.POINTER(c_int64)]),
    "vd_rows_to_planes": (c_int, [c_int, c_int64, c_int, P, c_int64, P, c_int64, P]),
    "vd_planes_to_rows": (c_int, [c_int, c_int64, c_int, P, c_int64, P, c_int64, P]),
}

_lib = None


def load():
    """Load (once) and type the in-tree shared library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__; __graft_entry__.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    lib.vdi_model_fingerprint.restype = c_uint64
    lib.vdi_model_fingerprint.argtypes = [P]
    _lib = lib
    return lib

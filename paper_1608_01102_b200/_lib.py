"""ctypes binding of libsmk.so (the C-ABI declared in include/smk.h).

The product path has no CPU fallback: importing a compute entry point without
the built library, or calling it without a CUDA device, raises.
"""

import ctypes
import os

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsmk.so")
if os.environ.get("SMK_LIB_VARIANT"):   # tuning builds (build.py --variant), never the product default
    LIB_PATH = os.path.join(HERE, f"libsmk_{os.environ['SMK_LIB_VARIANT']}.so")

SMK_OK = 0
SMK_NONCONVERGENCE = 1
SMK_TRUNCATION_OVERFLOW = 2
SMK_SINGULAR_BLOCK = 3
SMK_MAX_ITERATIONS = 4
SMK_ERR_ARG = -1
SMK_ERR_CUDA = -2

SMK_NEUMANN = 0
SMK_PERIODIC = 1
SMK_F64 = 0
SMK_F32 = 1


class smk_grid(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("res", ctypes.c_int * 3), ("h", ctypes.c_double),
                ("boundary", ctypes.c_int), ("dtype", ctypes.c_int)]


class smk_nso_params(ctypes.Structure):
    _fields_ = [("n_frames", ctypes.c_int), ("n_levels", ctypes.c_int), ("dt", ctypes.c_double),
                ("K", ctypes.c_double), ("r", ctypes.c_double), ("omega", ctypes.c_double),
                ("nu1", ctypes.c_int), ("nu2", ctypes.c_int), ("n_coarse", ctypes.c_int),
                ("color_mod", ctypes.c_int), ("t0", ctypes.c_int), ("n_total", ctypes.c_int),
                ("red_black", ctypes.c_int)]


VP3 = ctypes.c_void_p * 3


class smk_state(ctypes.Structure):
    _fields_ = [("V", VP3), ("PB", ctypes.c_void_p), ("U", VP3), ("P", ctypes.c_void_p)]


class smk_residual(ctypes.Structure):
    _fields_ = [("R1", VP3), ("R2", ctypes.c_void_p), ("R3", VP3), ("R4", ctypes.c_void_p)]


P = ctypes.c_void_p
I = ctypes.c_int
D = ctypes.c_double
PI = ctypes.POINTER(ctypes.c_int)
PD = ctypes.POINTER(ctypes.c_double)
G = ctypes.POINTER(smk_grid)
PP = ctypes.POINTER(smk_nso_params)
PS = ctypes.POINTER(smk_state)
PR = ctypes.POINTER(smk_residual)
I64 = ctypes.c_int64

# name -> (restype, argtypes)
SIGNATURES = {
    "smk_last_error": (ctypes.c_char_p, []),
    "smk_version": (I, []),
    "smk_launch_count": (ctypes.c_longlong, []),
    "smk_pool_trim": (None, []),
    "smk_div": (I, [G, I, P, P, P]),
    "smk_grad": (I, [G, I, P, P, P]),
    "smk_zero_walls": (I, [G, I, P, P]),
    "smk_laplacian": (I, [G, I, P, P, P]),
    "smk_inf_norm": (I, [I, P, I64, PD, P]),
    "smk_dot": (I, [I, P, P, I64, PD, P]),
    "smk_restrict_cell": (I, [G, I, P, P, P]),
    "smk_prolong_cell": (I, [G, I, P, P, I, P]),
    "smk_restrict_face": (I, [G, I, P, P, P]),
    "smk_prolong_face": (I, [G, I, P, P, I, P]),
    "smk_poisson_solve": (I, [G, P, P, D, I, PI, PD, P]),
    "smk_project": (I, [G, P, P, D, PI, PD, P]),
    "smk_transport_scalar": (I, [G, I, P, P, P, P]),
    "smk_advect": (I, [G, P, P, P, D, D, I, I, I, PI, PD, P]),
    "smk_scalar_stencil_v_adjoint": (I, [G, I, P, P, P, P]),
    "smk_advect_v_T": (I, [G, P, P, P, P, D, I, P]),
    "smk_transport_face": (I, [G, I, P, P, P, P]),
    "smk_self_adv_jac": (I, [G, I, P, P, P, P]),
    "smk_self_adv_jac_T": (I, [G, I, P, P, P, P]),
    "smk_semi_lagrangian": (I, [G, P, P, P, D, P]),
    "smk_sim_step": (I, [G, P, P, P, D, I, D, D, I, P, P, P, PI, PD, P]),
    "smk_kkt_residual": (I, [G, PP, PS, P, P, PR, PR, P]),
    "smk_scgs_sweep": (I, [G, PP, PS, P, P, PR, P]),
    "smk_nso_create": (P, [G, PP]),
    "smk_nso_destroy": (None, [P]),
    "smk_nso_levels": (I, [P]),
    "smk_nso_profile": (I, [P, I]),
    "smk_nso_profile_read": (I, [P, I, PD, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_longlong)]),
    "smk_nso_profile_read_level": (I, [P, I, I, PD, ctypes.POINTER(ctypes.c_longlong),
                                       ctypes.POINTER(ctypes.c_longlong)]),
    "smk_nso_device_bytes": (I64, [P]),
    "smk_nso_payload_values": (I64, [P]),
    "smk_nso_set_guide": (I, [P, P, P, P]),
    "smk_nso_set_K": (I, [P, D]),
    "smk_nso_vcycle": (I, [P, PS, P]),
    "smk_nso_residual_norms": (I, [P, PS, PD, PD, P]),
    "smk_nso_gauge_fix": (I, [P, PS, P]),
    "smk_nso_solve": (I, [P, PS, D, I, I, PI, PD, P]),
    "smk_nso_n_colors": (I, [P]),
    "smk_nso_level_residual": (I, [P, I, PS, P, P, P, PR, PR, P]),
    "smk_nso_level_color_pass": (I, [P, I, I, PS, P, P, P, PR, P]),
    "smk_axpby": (I, [I, P, P, D, D, I64, P]),
    "smk_axis_filter": (I, [I, I64, I, I64, P, I, D, D, P, P, P]),
    "smk_nccl_unique_id": (I, [P, I]),
    "smk_slabs_create": (P, [G, PP, I, I, I, I, I, P]),
    "smk_slabs_destroy": (None, [P]),
    "smk_slabs_levels": (I, [P]),
    "smk_slabs_device_bytes": (I64, [P]),
    "smk_slabs_frames": (I, [P, I, PI, PI]),
    "smk_slabs_set_guide": (I, [P, P, P, P]),
    "smk_slabs_vcycle": (I, [P, PS, P]),
    "smk_slabs_gauge_fix": (I, [P, PS, P]),
    "smk_slabs_residual_norms": (I, [P, PS, PD, PD, P]),
    "smk_slabs_profile": (I, [P, I]),
    "smk_slabs_profile_read_level": (I, [P, I, I, PD, ctypes.POINTER(ctypes.c_longlong),
                                         ctypes.POINTER(ctypes.c_longlong)]),
}

_lib = None


def load(path=LIB_PATH):
    """Load (once) and type the library.  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise errors.ExtensionMissing(
            f"{path} not built: run `python -m paper_1608_01102_b200.build` "
            "(the product path has no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (rt, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = rt
        fn.argtypes = args
    _lib = lib
    return lib


def last_error():
    msg = load().smk_last_error()
    return msg.decode() if msg else ""


def check(rc, what="", **info):
    """Map a status code onto the reference exception taxonomy (errors.py:4-56)."""
    if rc == SMK_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == SMK_NONCONVERGENCE:
        raise errors.NonConvergence(msg, residual=info.get("residual"), context=info.get("context"))
    if rc == SMK_TRUNCATION_OVERFLOW:
        raise errors.TruncationOverflow(msg, k_cap=info.get("k_cap"),
                                        last_term_norm=info.get("last_term_norm"))
    if rc == SMK_SINGULAR_BLOCK:
        raise errors.SingularBlock(msg)
    if rc == SMK_MAX_ITERATIONS:
        raise errors.MaxIterations(msg, result=info.get("result"))
    if rc == SMK_ERR_ARG:
        raise ValueError(msg)
    raise errors.DeviceError(msg)


def ptrs(tensors, n=3):
    """Array of `n` void* from a sequence of tensors (missing -> NULL)."""
    arr = (ctypes.c_void_p * n)()
    for i, t in enumerate(tensors):
        arr[i] = t.data_ptr() if t is not None else None
    return arr

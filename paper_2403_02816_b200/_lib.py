"""ctypes binding of the C-ABI library `_lib/libcglb200.so` (include/cgl_b200.h).

There is no CPU fallback: loading fails loudly when the library is missing,
and every compute entry point requires CUDA tensors.  Tensors are torch
complex128 CUDA tensors, C-contiguous; work is enqueued on torch's current
stream.
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import _build

_LIB = None

c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_ptr = ctypes.c_void_p
c_int = ctypes.c_int
c_u64 = ctypes.c_uint64

# CGL_* reason codes (include/cgl_b200.h) -> reference reason strings
REASONS = {
    0: "finite-time blow-up in cubic flow",      # flows.py:95-96
    1: "non-finite cubic flow output",           # flows.py:99-100
    2: "finite-time blow-up in quintic flow",    # flows.py:111-112
    3: "non-finite quintic flow output",         # flows.py:114-115
    4: "non-finite RK4 flow output",             # flows.py:131-132
    5: "non-finite state",                       # integrators.py:274-278
}
NONFINITE_STATE = 5
NO_DIVERGENCE = (1 << 64) - 1
POS_DEVICE = 1 << 63

STAGE = {"if4_pre": 0, "if4_mid": 1, "if4_end": 2, "flow1": 3, "flow2": 4, "split4_mid": 5,
         "split4_end": 6, "strang_end": 7, "if2_pre": 8, "if2_end": 9, "fif4_s1": 10, "fif4_s2": 11,
         "fif4_s3": 12, "fif4_s4": 13, "flow_end": 14, "if4_midq": 17,
         "if4_endq": 18}


def new_flag(base=0):
    """Device flag record (cgl_flag_t): key = all ones, step base, done = 0."""
    f = torch.zeros(3, dtype=torch.int64, device="cuda")
    f[0] = -1
    f[1] = base
    return f


def rel_pos(local_step):
    """Device-relative position of local step `local_step` (>= 1) of a chunk."""
    return POS_DEVICE | (int(local_step) << 24)


def flag_advance(flag, n):
    check(load().cgl_flag_advance(stream(), flag_ptr(flag), int(n)), "cgl_flag_advance")

KIND_CODES = {"cubic": 0, "cubic_quintic": 1, "coupled_cubic_quintic": 2}


class Nonlinear(ctypes.Structure):
    _fields_ = [("alpha3", c_dbl), ("beta3", c_dbl), ("alpha4", c_dbl),
                ("beta4", c_dbl), ("alpha5", c_dbl), ("kind", c_int)]


class FftOps(ctypes.Structure):
    """cgl_fft_ops_t (include/cgl_b200.h): operands of a fused pencil-FFT pass."""
    _fields_ = [("u", c_ptr), ("u_out", c_ptr), ("g", c_ptr * 3), ("g_out", c_ptr), ("tables", (c_ptr * 3) * 2),
                ("tau", c_dbl), ("scale", c_dbl), ("nl", Nonlinear), ("flag", c_ptr), ("pos", c_u64)]


FFT_PROGRAMS = {"plain": 0, "if4_start": 1, "if4_b1": 2, "if4_b2": 3, "if4_b3": 4, "if4_b4": 5, "g": 6,
                "str_start": 7, "str_a0": 8, "str_mid": 9, "str_a0f": 10}

_SIGS = {
    "cgl_version": (ctypes.c_char_p, []),
    "cgl_last_error": (ctypes.c_char_p, []),
    "cgl_abi_version": (c_int, []),
    "cgl_launch_count": (ctypes.c_ulonglong, []),
    "cgl_probe_dmma": (c_dbl, [c_ptr, c_int]),
    "cgl_zgemm": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_i64, c_ptr, c_i64, c_i64,
                          c_ptr, c_i64, c_i64, c_i64, c_dbl, c_dbl, c_ptr, c_i64, c_i64, c_dbl,
                          c_ptr, c_u64]),
    "cgl_mode_product": (c_int, [c_ptr, c_int, c_ptr, c_int, c_ptr, c_ptr, c_i64, c_ptr, c_ptr,
                                 c_dbl, c_ptr, c_dbl, c_ptr, c_u64]),
    "cgl_mode_product_batch": (c_int, [c_ptr, c_int, c_ptr, c_int, c_int, c_ptr, c_ptr, c_i64, c_ptr, c_ptr,
                                       c_dbl, c_ptr, c_dbl, c_ptr, c_u64]),
    "cgl_tucker": (c_int, [c_ptr, c_int, c_ptr, c_int, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_u64]),
    "cgl_oz_slice_bytes": (c_i64, [c_int, c_i64, c_i64, c_int]),
    "cgl_oz_slice": (c_int, [c_ptr, c_int, c_ptr, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_ptr, c_i64,
                             c_ptr, c_i64]),
    "cgl_oz_gemm": (c_int, [c_ptr, c_int, c_i64, c_i64, c_i64, c_int, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                            c_ptr, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_ptr, c_u64]),
    "cgl_oz_slice_multi": (c_int, [c_ptr, c_int, c_int, c_ptr, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_int,
                                   c_ptr, c_i64, c_ptr, c_i64]),
    "cgl_oz_trace": (c_int, [c_ptr]),
    "cgl_prof_set": (c_int, [c_ptr, c_ptr, ctypes.c_uint]),
    "cgl_oz_geometry": (c_int, [ctypes.POINTER(c_int), ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
    "cgl_oz_gemm_t": (c_int, [c_ptr, c_int, c_i64, c_i64, c_i64, c_int, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                              c_ptr, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_ptr, c_u64]),
    "cgl_oz_zmap": (c_int, [c_ptr, c_int, c_ptr, c_i64, c_i64, c_int, c_ptr]),
    "cgl_uniforms": (c_int, [c_ptr, c_u64, c_u64, c_i64, c_ptr]),
    "cgl_seeded_ic": (c_int, [c_ptr, c_int, c_u64, c_int, c_ptr, c_ptr, c_ptr]),
    "cgl_stage_slice": (c_int, [c_ptr, c_int, c_i64, c_i64, c_ptr, c_dbl, c_dbl, c_ptr, c_ptr, c_ptr, c_u64, c_ptr,
                                c_ptr]),
    "cgl_lincomb": (c_int, [c_ptr, c_i64, c_int, c_ptr, c_ptr, c_ptr, c_ptr, c_u64]),
    "cgl_eval_g": (c_int, [c_ptr, c_i64, c_ptr, c_int, c_ptr, c_dbl, c_ptr, c_ptr, c_u64]),
    "cgl_cubic_flow": (c_int, [c_ptr, c_i64, c_dbl, c_ptr, c_ptr, c_dbl, c_ptr, c_ptr, c_u64]),
    "cgl_quintic_flow": (c_int, [c_ptr, c_i64, c_dbl, c_ptr, c_ptr, c_dbl, c_ptr, c_ptr, c_u64]),
    "cgl_rk4_flow": (c_int, [c_ptr, c_i64, c_dbl, c_ptr, c_int, c_ptr, c_dbl, c_ptr, c_ptr, c_u64]),
    "cgl_check_finite": (c_int, [c_ptr, c_i64, c_int, c_ptr, c_ptr, c_u64]),
    "cgl_flag_reset": (c_int, [c_ptr, c_ptr]),
    "cgl_flag_advance": (c_int, [c_ptr, c_ptr, ctypes.c_ulonglong]),
    "cgl_stage": (c_int, [c_ptr, c_int, c_int, c_i64, c_ptr, c_dbl, c_dbl, c_ptr, c_ptr, c_ptr, c_u64]),
    "cgl_stage_fourier": (c_int, [c_ptr, c_int, c_int, c_int, c_ptr, c_ptr, c_dbl, c_dbl, c_ptr, c_ptr, c_ptr,
                                  c_ptr, c_u64]),
    "cgl_stage_fourier_cols": (c_int, [c_ptr, c_int, c_int, c_int, c_ptr, c_i64, c_i64, c_ptr, c_dbl, c_dbl, c_ptr,
                                       c_ptr, c_ptr, c_ptr, c_u64]),
    "cgl_separable_mul_cols": (c_int, [c_ptr, c_int, c_ptr, c_i64, c_i64, c_ptr, c_dbl, c_ptr, c_ptr, c_ptr, c_u64]),
    "cgl_fft_plan_many": (c_int, [c_int, c_ptr, c_i64, c_i64, c_i64, c_i64, c_i64, ctypes.POINTER(c_ptr)]),
    "cgl_pointwise_mul": (c_int, [c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_u64]),
    "cgl_symbol_exp": (c_int, [c_ptr, c_i64, c_dbl, c_ptr, c_ptr]),
    "cgl_separable_mul": (c_int, [c_ptr, c_int, c_ptr, c_ptr, c_dbl, c_ptr, c_ptr, c_ptr, c_u64]),
    "cgl_fft_plan": (c_int, [c_int, c_ptr, ctypes.POINTER(c_ptr)]),
    "cgl_fft_exec": (c_int, [c_ptr, c_ptr, c_ptr, c_ptr, c_int]),
    "cgl_fft_destroy": (c_int, [c_ptr]),
    "cgl_fft_pass_supported": (c_int, [c_int, c_ptr]),
    "cgl_tucker2d": (c_int, [c_ptr, c_int, c_int, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                             c_dbl, c_ptr, c_u64]),
    "cgl_slab_pack": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr]),
    "cgl_slab_unpack": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr]),
    "cgl_slab_transpose": (c_int, [c_ptr, c_ptr, c_int, c_int, c_i64, c_i64, c_ptr, c_ptr, c_ptr]),
    "cgl_fft_pass": (c_int, [c_ptr, c_int, c_int, c_ptr, c_int, c_int, c_ptr, c_ptr, ctypes.POINTER(FftOps)]),
    "cgl_rk_stage": (c_int, [c_ptr, c_int, c_ptr, c_int, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                             c_dbl, c_dbl, c_int, c_ptr, c_u64]),
}

EXPORTED = tuple(_SIGS)


def lib_path():
    return _build.LIB


def load():
    """Load (building first if sources changed and nvcc is present)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = _build.LIB
    override = os.environ.get("CGL_LIB_OVERRIDE")  # kernel A/B experiments (tools/oz_bench.py)
    if override:
        path = override
    elif not os.path.exists(path) or _build.needs_build():
        try:
            _build.build()
        except (RuntimeError, FileNotFoundError) as e:
            if not os.path.exists(path):
                raise ImportError(f"cgl_b200 CUDA library missing and cannot be built: {e}") from e
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        if override and not hasattr(lib, name):
            continue  # A/B variant libraries may predate newer entry points
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


class CglError(RuntimeError):
    pass


def check(rc, what):
    if rc != 0:
        msg = load().cgl_last_error().decode(errors="replace")
        if rc == -2:
            raise ValueError(f"{what}: {msg}")
        raise CglError(f"{what} failed (rc={rc}): {msg}")


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2403_02816_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")


def stream():
    return c_ptr(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return c_ptr(t.data_ptr()) if t is not None else c_ptr(0)


def ptr_array(ts):
    arr = (c_ptr * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = t.data_ptr() if t is not None else 0
    return arr


def i64_array(vals):
    arr = (c_i64 * len(vals))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr


def dbl_array(vals):
    arr = (c_dbl * len(vals))()
    for i, v in enumerate(vals):
        arr[i] = float(v)
    return arr


def nonlinear_struct(kind, params):
    return Nonlinear(params.alpha3, params.beta3, params.alpha4, params.beta4,
                     params.alpha5, KIND_CODES[kind])


def flag_ptr(flag):
    return c_ptr(flag.data_ptr()) if flag is not None else c_ptr(0)

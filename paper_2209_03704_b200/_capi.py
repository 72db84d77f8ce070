"""ctypes binding of the C ABI in include/segconv_b200.h.

Loads the in-tree ``libsegconv_b200.so`` (built by ``paper_2209_03704_b200.build``).
There is no fallback: if the library is missing or cannot be loaded, importing
the package's compute entry points raises ``SegconvLibraryError``.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libsegconv_b200.so")

# segconv_status
OK, E_SHAPE, E_CONTRACT, E_CUDA, E_UNSUPPORTED, E_IO, E_PARSE, E_NCCL = range(8)
# segconv_dtype
F32, F64, BF16, F16_SPLIT = 0, 1, 2, 3
# segconv_math
MATH_AUTO, MATH_FFMA, MATH_EXACT, MATH_BF16, MATH_TF32, MATH_F16X3 = range(6)
# epilogue flags
EPI_NONE, EPI_BIAS, EPI_RELU, EPI_TANH = 0, 1, 2, 4
# panel layouts
PANEL_REF, PANEL_KMAJOR, PANEL_UMMA, PANEL_UMMA_FOLD = 0, 1, 2, 3


class SegconvLibraryError(RuntimeError):
    pass


class Geometry(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("n_in", "kh", "kw", "p_orig", "p_fused", "up_h", "up_w",
                                       "out_h", "out_w", "trim_extra_row", "trim_extra_col")]


class SubKernels(C.Structure):
    _fields_ = [
        ("source_kh", C.c_int), ("source_kw", C.c_int), ("p_orig", C.c_int),
        ("p_orig_parity", C.c_int), ("cin", C.c_int), ("cout", C.c_int), ("cout_pad", C.c_int),
        ("sub_kh", C.c_int * 4), ("sub_kw", C.c_int * 4), ("off_r", C.c_int * 4),
        ("off_c", C.c_int * 4), ("u0", C.c_int * 4), ("v0", C.c_int * 4),
        ("sub_offset", C.c_int64 * 4), ("total_elems", C.c_int64), ("dtype", C.c_int),
        ("layout", C.c_int), ("n_tile", C.c_int), ("k_block", C.c_int), ("math", C.c_int),
    ]


class TensorFileInfo(C.Structure):
    _fields_ = [("height", C.c_int), ("width", C.c_int), ("channels", C.c_int),
                ("precision", C.c_int)]


class Layer(C.Structure):
    """segconv_layer: one layer of a multi-GPU stack."""
    _fields_ = [("n_in", C.c_int), ("cin", C.c_int), ("cout", C.c_int), ("kh", C.c_int), ("kw", C.c_int),
                ("p_orig", C.c_int), ("h_kernel", C.c_void_p), ("kernel_dtype", C.c_int),
                ("h_bias", C.c_void_p), ("epilogue", C.c_uint), ("math", C.c_int)]


class Timing(C.Structure):
    _fields_ = [("n_gpus", C.c_int), ("h2d_ms", C.c_double), ("compute_ms", C.c_double),
                ("gather_ms", C.c_double), ("d2h_ms", C.c_double), ("total_ms", C.c_double)]


# (name, restype, argtypes) for every symbol include/segconv_b200.h declares.
_vp, _i, _u, _sz = C.c_void_p, C.c_int, C.c_uint, C.c_size_t
SIGNATURES = {
    "segconv_tconv_geometry": (_i, [_i, _i, _i, _i, C.POINTER(Geometry)]),
    "segconv_first_active_tap": (_i, [_i, _i]),
    "segconv_active_tap_count": (_i, [_i, _i, _i]),
    "segconv_class_input_offset": (_i, [_i, _i]),
    "segconv_subkernels_init": (_i, [_i, _i, _i, _i, _i, _i, _i, C.POINTER(SubKernels)]),
    "segconv_subkernels_for_math": (_i, [_i, _i, _i, _i, _i, _i, _i, C.POINTER(SubKernels)]),
    "segconv_segregate": (_i, [_vp, _i, C.POINTER(SubKernels), _vp, _vp]),
    "segconv_transpose_conv_fused": (_i, [_vp, _i, _i, _i, _i, C.POINTER(SubKernels), _vp,
                                          C.POINTER(Geometry), _vp, _u, _i, _vp, _i, _vp]),
    "segconv_transpose_conv_fused_host": (_i, [_vp, _vp, _i, _i, _i, _i, C.POINTER(SubKernels),
                                               _vp, C.POINTER(Geometry), _vp, _u, _i, _vp, _vp,
                                               _i, _i, _vp]),
    "segconv_transpose_conv_fused_backward": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _i, _i, _i,
                                                   _i, _i, _vp, _vp, _i, _vp]),
    "segconv_select_math": (_i, [_i, _i, _i, _i, _i, _i]),
    "segconv_peek_tensor_file": (_i, [C.c_char_p, C.POINTER(TensorFileInfo)]),
    "segconv_load_tensor": (_i, [C.c_char_p, _i, _vp, _sz]),
    "segconv_save_tensor": (_i, [C.c_char_p, _vp, _i, _i, _i, _i]),
    "segconv_load_tensor_batch": (_i, [C.POINTER(C.c_char_p), _i, _i, _vp, _vp, _vp]),
    "segconv_last_error_offset": (_sz, []),
    "segconv_upsample2x_pad": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _vp]),
    "segconv_upsample2x_pad_backward": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _vp]),
    "segconv_conv2d_valid": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _i, _i, _i, _vp, _u, _i, _vp, _vp]),
    "segconv_conv2d_valid_backward": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _vp, _i, _i, _i, _i, _vp,
                                           _vp, _i, _vp]),
    "segconv_naive_workspace_bytes": (_sz, [_i, _i, _i, _i, _i]),
    "segconv_transpose_conv_naive": (_i, [_vp, _i, _i, _i, _i, _vp, _i, _i, _i, _i, _vp, _sz,
                                          _vp, _u, _i, _vp, _vp]),
    "segconv_count_ops": (_i, [_i, _i, _i, _i, _i, _i, C.POINTER(C.c_uint64)]),
    "segconv_stack_create": (_i, [C.POINTER(Layer), _i, _i, _i, _i, C.POINTER(_vp)]),
    "segconv_stack_forward": (_i, [_vp, _vp, _i, _vp, C.POINTER(Timing)]),
    "segconv_stack_output": (_vp, [_vp, _i]),
    "segconv_stack_gpus": (_i, [_vp]),
    "segconv_stack_destroy": (None, [_vp]),
    "segconv_stack_run": (_i, [C.POINTER(Layer), _i, _i, _vp, _i, _i, _vp, C.POINTER(Timing)]),
    "segconv_last_error": (C.c_char_p, []),
    "segconv_last_path": (C.c_char_p, []),
    "segconv_version": (C.c_char_p, []),
    "segconv_launch_count": (C.c_uint64, []),
    "segconv_debug_trace": (_sz, [_vp, _sz]),
    "segconv_debug_wide_schedule": (_sz, [C.POINTER(C.c_longlong), C.POINTER(C.c_int), _i, C.c_longlong, _i,
                                          C.POINTER(C.c_uint16), _sz]),
}

_lib = None


def lib():
    """The loaded C library (raises SegconvLibraryError if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SegconvLibraryError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2209_03704_b200.build` "
                "(there is no CPU fallback)")
        try:
            L = C.CDLL(LIB_PATH)
        except OSError as e:  # pragma: no cover
            raise SegconvLibraryError(f"cannot load {LIB_PATH}: {e}") from e
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return (lib().segconv_last_error() or b"").decode()

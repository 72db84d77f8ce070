"""ctypes wrappers over the CPU oracle and the reference shim (test infrastructure)."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsegconv_ref.so")

__all__ = [
    "Geometry", "load_oracle", "load_ref", "ref_available", "geometry", "first_active_tap",
    "active_tap_count", "class_input_offset", "subkernel_dims", "segregate", "tconv_fused",
    "tconv_naive", "scatter_f64", "count_ops", "ref_geometry", "ref_segregate", "ref_tconv_fused",
    "ref_tconv_naive", "ref_tconv_fused_parallel", "ref_run_verify", "ref_verify_case",
    "ref_count_ops", "ref_time_fused_batch", "OracleError", "bf16_round", "tf32_round",
    "tconv_backward", "scatter_backward_f64", "ref_tconv_backward", "ref_time_backward",
    "ref_save_tensor", "ref_load_tensor", "conv2d_valid", "ref_conv2d_valid",
    "conv2d_valid_backward", "ref_conv2d_valid_backward",
]


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


_P = np.ctypeslib.ndpointer
_lib = None
_ref = None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def load_oracle():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            raise OracleError(-1, f"{ORACLE_SO} missing: run `make -C oracle oracle`")
        lib = C.CDLL(ORACLE_SO)
        ip = C.POINTER(C.c_int)
        lib.orc_tconv_geometry.argtypes = [C.c_int] * 4 + [ip]
        for name, T in (("f32", C.c_float), ("f64", C.c_double)):
            pt = C.POINTER(T)
            for op in ("fused", "naive"):
                fn = getattr(lib, f"orc_tconv_{op}_{name}")
                fn.argtypes = [pt, C.c_int, C.c_int, C.c_int, pt, C.c_int, C.c_int, C.c_int,
                               C.c_int, pt]
            seg = getattr(lib, f"orc_segregate_{name}")
            seg.argtypes = [pt, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, pt]
            seg.restype = C.c_size_t
        lib.orc_scatter_f64.argtypes = lib.orc_tconv_fused_f64.argtypes
        for name, T in (("f32", C.c_float), ("f64", C.c_double)):
            pt = C.POINTER(T)
            getattr(lib, f"orc_tconv_backward_{name}").argtypes = [
                pt, C.c_int, C.c_int, C.c_int, pt, C.c_int, C.c_int, C.c_int, C.c_int, pt, pt, pt]
        lib.orc_scatter_backward_f64.argtypes = lib.orc_tconv_backward_f64.argtypes
        for name, T in (("f32", C.c_float), ("f64", C.c_double)):
            pt = C.POINTER(T)
            getattr(lib, f"orc_conv2d_valid_backward_{name}").argtypes = [pt] + [C.c_int] * 4 + \
                [pt] + [C.c_int] * 3 + [pt, pt, pt]
            getattr(lib, f"orc_conv2d_valid_{name}").argtypes = [pt] + [C.c_int] * 4 + [pt] + \
                [C.c_int] * 3 + [pt]
        lib.orc_subkernel_dims.argtypes = [C.c_int, C.c_int, C.c_int, ip, ip]
        lib.orc_count_ops.argtypes = [C.c_int] * 6 + [C.POINTER(C.c_uint64)]
        _lib = lib
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def load_ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise OracleError(-1, f"{REF_SO} missing: run `make -C oracle ref` where "
                              "/root/reference exists")
        lib = C.CDLL(REF_SO)
        fp, dp, ip = C.POINTER(C.c_float), C.POINTER(C.c_double), C.POINTER(C.c_int)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_tconv_geometry.argtypes = [C.c_int] * 4 + [ip]
        lib.ref_segregate_f32.argtypes = [fp] + [C.c_int] * 5 + [fp, ip, ip]
        for nm, T in (("f32", fp), ("f64", dp)):
            for op in ("fused", "naive"):
                getattr(lib, f"ref_tconv_{op}_{nm}").argtypes = [
                    T, C.c_int, C.c_int, C.c_int, T, C.c_int, C.c_int, C.c_int, C.c_int, T]
        for nm, T in (("f32", fp), ("f64", dp)):
            getattr(lib, f"ref_tconv_backward_{nm}").argtypes = [
                T, C.c_int, C.c_int, C.c_int, T, C.c_int, C.c_int, C.c_int, C.c_int, T, T, T]
        lib.ref_time_backward_f32.argtypes = [
            fp, C.c_int, C.c_int, C.c_int, fp, C.c_int, C.c_int, C.c_int, C.c_int, fp, C.c_int,
            fp, fp, dp]
        lib.ref_conv2d_valid_f32.argtypes = [fp] + [C.c_int] * 4 + [fp] + [C.c_int] * 3 + [fp]
        for nm, T in (("f32", fp), ("f64", dp)):
            getattr(lib, f"ref_conv2d_valid_backward_{nm}").argtypes = [T] + [C.c_int] * 4 + [T] + \
                [C.c_int] * 3 + [T, T, T]
        lib.ref_save_tensor.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]
        lib.ref_load_tensor.argtypes = [C.c_char_p, C.c_int, C.c_void_p, C.c_size_t, ip]
        lib.ref_last_error_offset.restype = C.c_size_t
        lib.ref_tconv_fused_parallel_f32.argtypes = [
            fp, C.c_int, C.c_int, C.c_int, fp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, fp]
        lib.ref_count_ops.argtypes = [C.c_int] * 6 + [C.POINTER(C.c_uint64)]
        lib.ref_run_verify.argtypes = [C.c_int, C.c_uint64, C.c_int, ip]
        lib.ref_verify_case.argtypes = [C.c_uint64, C.c_int, ip, fp, fp, fp]
        lib.ref_time_fused_batch_f32.argtypes = [
            C.c_int, fp, C.c_int, C.c_int, C.c_int, fp, C.c_int, C.c_int, C.c_int, C.c_int,
            C.c_int, fp, dp]
        _ref = lib
    return _ref


def _ptr(a, T):
    return a.ctypes.data_as(C.POINTER(T))


def _check(code, lib=None):
    if code:
        msg = lib.ref_last_error().decode() if lib is not None and lib is _ref else ""
        raise OracleError(code, msg)


@dataclass(frozen=True)
class Geometry:
    n_in: int
    kh: int
    kw: int
    p_orig: int
    p_fused: int
    up_h: int
    up_w: int
    out_h: int
    out_w: int
    trim_extra_row: bool
    trim_extra_col: bool


# ----------------------------------------------------------------- plain-C port
def geometry(n_in, kh, kw, p):
    g = (C.c_int * 11)()
    _check(load_oracle().orc_tconv_geometry(n_in, kh, kw, p, g))
    v = list(g)
    return Geometry(*v[:9], bool(v[9]), bool(v[10]))


def first_active_tap(p, r):
    return load_oracle().orc_first_active_tap(p, r)


def active_tap_count(n, p, r):
    return load_oracle().orc_active_tap_count(n, p, r)


def class_input_offset(p, r):
    return load_oracle().orc_class_input_offset(p, r)


def subkernel_dims(kh, kw, p):
    d, o = (C.c_int * 8)(), (C.c_int * 8)()
    load_oracle().orc_subkernel_dims(kh, kw, p, d, o)
    return [(d[2 * q], d[2 * q + 1]) for q in range(4)], [(o[2 * q], o[2 * q + 1]) for q in range(4)]


def segregate(k, p):
    """Concatenated sub-kernels, class order r*2+c (returns list of 4 arrays)."""
    k = np.asarray(k)
    f64 = k.dtype == np.float64
    k = _f64(k) if f64 else _f32(k)
    kh, kw, cin, cout = k.shape
    T = C.c_double if f64 else C.c_float
    out = np.empty(k.size, dtype=k.dtype)
    fn = load_oracle().orc_segregate_f64 if f64 else load_oracle().orc_segregate_f32
    fn(_ptr(k, T), kh, kw, cin, cout, p, _ptr(out, T))
    dims, _ = subkernel_dims(kh, kw, p)
    subs, off = [], 0
    for (a, b) in dims:
        n = a * b * cin * cout
        subs.append(out[off:off + n].reshape(a, b, cin, cout))
        off += n
    return subs


def _run(op, x, k, p, lib_fn_prefix, lib):
    x = np.asarray(x)
    f64 = x.dtype == np.float64
    x = _f64(x) if f64 else _f32(x)
    k = _f64(k) if f64 else _f32(k)
    squeeze = x.ndim == 3
    if squeeze:
        x = x[None]
    b, n, n2, cin = x.shape
    kh, kw, kc, cout = k.shape
    g = geometry(n, kh, kw, p)
    out = np.empty((b, g.out_h, g.out_w, cout), dtype=x.dtype)
    T = C.c_double if f64 else C.c_float
    fn = getattr(lib, f"{lib_fn_prefix}_{op}_{'f64' if f64 else 'f32'}")
    _check(fn(_ptr(x, T), b, n, cin, _ptr(k, T), kh, kw, cout, p, _ptr(out, T)), lib)
    return out[0] if squeeze else out


def tconv_fused(x, k, p):
    """Segregated transpose conv (batch NHWC or single HWC), reference accumulation order."""
    return _run("fused", x, k, p, "orc_tconv", load_oracle())


def tconv_naive(x, k, p):
    return _run("naive", x, k, p, "orc_tconv", load_oracle())


def scatter_f64(x, k, p):
    x, k = _f64(x), _f64(k)
    squeeze = x.ndim == 3
    if squeeze:
        x = x[None]
    b, n, _, cin = x.shape
    kh, kw, _, cout = k.shape
    g = geometry(n, kh, kw, p)
    out = np.empty((b, g.out_h, g.out_w, cout))
    _check(load_oracle().orc_scatter_f64(_ptr(x, C.c_double), b, n, cin, _ptr(k, C.c_double),
                                         kh, kw, cout, p, _ptr(out, C.c_double)))
    return out[0] if squeeze else out


def _backward(fn_name, x, k, p, gy, lib, force_f64=False):
    x = np.asarray(x)
    f64 = force_f64 or x.dtype == np.float64
    cast = _f64 if f64 else _f32
    x, k, gy = cast(x), cast(k), cast(gy)
    squeeze = x.ndim == 3
    if squeeze:
        x, gy = x[None], gy[None]
    b, n, _, cin = x.shape
    kh, kw, _, cout = k.shape
    g = geometry(n, kh, kw, p)
    if gy.shape != (b, g.out_h, g.out_w, cout):
        raise OracleError(2, f"output gradient shape {gy.shape} != {(b, g.out_h, g.out_w, cout)}")
    gx = np.empty_like(x)
    gk = np.empty_like(k)
    T = C.c_double if f64 else C.c_float
    fn = getattr(lib, fn_name if force_f64 else f"{fn_name}_{'f64' if f64 else 'f32'}")
    _check(fn(_ptr(x, T), b, n, cin, _ptr(k, T), kh, kw, cout, p, _ptr(gy, T), _ptr(gx, T),
              _ptr(gk, T)), lib)
    return (gx[0] if squeeze else gx), gk


def tconv_backward(x, k, p, gy):
    """(input grad, kernel grad) of the fused layer, reference order (layers.hpp:171-211);
    the kernel grad is summed over the batch."""
    return _backward("orc_tconv_backward", x, k, p, gy, load_oracle())


def scatter_backward_f64(x, k, p, gy):
    return _backward("orc_scatter_backward_f64", x, k, p, gy, load_oracle(), force_f64=True)


def _conv_valid(lib, prefix, src, k):
    src = np.asarray(src)
    f64 = src.dtype == np.float64 and prefix == "orc"
    cast = _f64 if f64 else _f32
    src, k = cast(src), cast(k)
    squeeze = src.ndim == 3
    if squeeze:
        src = src[None]
    b, h, w, cin = src.shape
    kh, kw, _, cout = k.shape
    out = np.empty((b, h - kh + 1, w - kw + 1, cout), dtype=src.dtype)
    T = C.c_double if f64 else C.c_float
    fn = getattr(lib, f"{prefix}_conv2d_valid_{'f64' if f64 else 'f32'}")
    _check(fn(_ptr(src, T), b, h, w, cin, _ptr(k, T), kh, kw, cout, _ptr(out, T)), lib)
    return out[0] if squeeze else out


def _conv_backward(lib, prefix, src, k, gy):
    src = np.asarray(src)
    f64 = src.dtype == np.float64
    cast = _f64 if f64 else _f32
    src, k, gy = cast(src), cast(k), cast(gy)
    squeeze = src.ndim == 3
    if squeeze:
        src, gy = src[None], gy[None]
    b, h, w, cin = src.shape
    kh, kw, _, cout = k.shape
    if gy.shape != (b, h - kh + 1, w - kw + 1, cout):
        raise OracleError(2, f"output gradient shape {gy.shape}")
    gx, gk = np.empty_like(src), np.empty_like(k)
    T = C.c_double if f64 else C.c_float
    fn = getattr(lib, f"{prefix}_conv2d_valid_backward_{'f64' if f64 else 'f32'}")
    _check(fn(_ptr(src, T), b, h, w, cin, _ptr(k, T), kh, kw, cout, _ptr(gy, T), _ptr(gx, T), _ptr(gk, T)), lib)
    return (gx[0] if squeeze else gx), gk


def conv2d_valid_backward(src, k, gy):
    """(input grad, kernel grad) of conv2d_valid, reference order (layers.hpp:98-122)."""
    return _conv_backward(load_oracle(), "orc", src, k, gy)


def ref_conv2d_valid_backward(src, k, gy):
    return _conv_backward(load_ref(), "ref", src, k, gy)


def conv2d_valid(src, k):
    """Valid correlation, reference order (reference_ops.hpp:86-102), batch or single map."""
    return _conv_valid(load_oracle(), "orc", src, k)


def ref_conv2d_valid(src, k):
    return _conv_valid(load_ref(), "ref", src, k)


def count_ops(n, cin, cout, kh, kw, p):
    """(naive_mults, naive_adds, fused_mults, fused_adds)."""
    o = (C.c_uint64 * 4)()
    _check(load_oracle().orc_count_ops(n, cin, cout, kh, kw, p, o))
    return tuple(int(v) for v in o)


# ------------------------------------------------------------ reference shim
def ref_geometry(n_in, kh, kw, p):
    g = (C.c_int * 11)()
    lib = load_ref()
    _check(lib.ref_tconv_geometry(n_in, kh, kw, p, g), lib)
    v = list(g)
    return Geometry(*v[:9], bool(v[9]), bool(v[10]))


def ref_segregate(k, p):
    k = _f32(k)
    kh, kw, cin, cout = k.shape
    lib = load_ref()
    out = np.empty(k.size, dtype=np.float32)
    d, o = (C.c_int * 8)(), (C.c_int * 8)()
    _check(lib.ref_segregate_f32(_ptr(k, C.c_float), kh, kw, cin, cout, p, _ptr(out, C.c_float),
                                 d, o), lib)
    subs, off = [], 0
    for q in range(4):
        a, b = d[2 * q], d[2 * q + 1]
        n = a * b * cin * cout
        subs.append(out[off:off + n].reshape(a, b, cin, cout))
        off += n
    return subs, [(o[2 * q], o[2 * q + 1]) for q in range(4)]


def ref_tconv_fused(x, k, p):
    return _run("fused", x, k, p, "ref_tconv", load_ref())


def ref_tconv_naive(x, k, p):
    return _run("naive", x, k, p, "ref_tconv", load_ref())


def ref_tconv_fused_parallel(x, k, p, workers):
    x, k = _f32(x), _f32(k)
    squeeze = x.ndim == 3
    if squeeze:
        x = x[None]
    b, n, _, cin = x.shape
    kh, kw, _, cout = k.shape
    g = geometry(n, kh, kw, p)
    out = np.empty((b, g.out_h, g.out_w, cout), dtype=np.float32)
    lib = load_ref()
    _check(lib.ref_tconv_fused_parallel_f32(_ptr(x, C.c_float), b, n, cin, _ptr(k, C.c_float), kh,
                                            kw, cout, p, workers, _ptr(out, C.c_float)), lib)
    return out[0] if squeeze else out


def ref_tconv_backward(x, k, p, gy):
    """The reference's own net::FusedTConv forward + backward per image."""
    return _backward("ref_tconv_backward", x, k, p, gy, load_ref())


def ref_time_backward(x, k, p, gy, workers):
    """Times the reference backward (threads over the batch); returns (gx, gk, seconds)."""
    x, k, gy = _f32(x), _f32(k), _f32(gy)
    b, n, _, cin = x.shape
    kh, kw, _, cout = k.shape
    gx, gk = np.empty_like(x), np.empty_like(k)
    secs = C.c_double()
    lib = load_ref()
    fp = C.c_float
    _check(lib.ref_time_backward_f32(_ptr(x, fp), b, n, cin, _ptr(k, fp), kh, kw, cout, p,
                                     _ptr(gy, fp), workers, _ptr(gx, fp), _ptr(gk, fp),
                                     C.byref(secs)), lib)
    return gx, gk, secs.value


def ref_save_tensor(path, t):
    """The reference's save_tensor (tensor_io.hpp:93-103) on an (h, w, c) f32/f64 array."""
    t = np.ascontiguousarray(t)
    f64 = t.dtype == np.float64
    t = _f64(t) if f64 else _f32(t)
    lib = load_ref()
    _check(lib.ref_save_tensor(os.fsencode(path), t.ctypes.data, *t.shape, int(f64)), lib)


def ref_load_tensor(path, f64=False):
    """The reference's load_tensor<T>; returns the array, or raises OracleError
    with .code (5 IoError, 6 ParseError, 2 ContractError) and .offset."""
    lib = load_ref()
    d = (C.c_int * 4)()
    cap = 1 << 22
    buf = np.empty(cap, dtype=np.float64 if f64 else np.float32)
    code = lib.ref_load_tensor(os.fsencode(path), int(f64), buf.ctypes.data, cap, d)
    if code:
        e = OracleError(code, (lib.ref_last_error() or b"").decode())
        e.offset = int(lib.ref_last_error_offset())
        raise e
    return buf[: d[0] * d[1] * d[2]].reshape(d[0], d[1], d[2]).copy()


def ref_count_ops(n, cin, cout, kh, kw, p):
    o = (C.c_uint64 * 4)()
    lib = load_ref()
    _check(lib.ref_count_ops(n, cin, cout, kh, kw, p, o), lib)
    return tuple(int(v) for v in o)


def ref_run_verify(cases=200, seed=20240911, inject_fault_case=-1):
    o = (C.c_int * 3)()
    lib = load_ref()
    _check(lib.ref_run_verify(cases, seed, inject_fault_case, o), lib)
    return {"cases_run": o[0], "failures": o[1], "first_failure": o[2]}


def ref_verify_case(seed, case_index):
    lib = load_ref()
    d = (C.c_int * 5)()
    xb = np.zeros(16 * 16 * 4, dtype=np.float32)
    kb = np.zeros(7 * 7 * 4 * 4, dtype=np.float32)
    yb = np.zeros(40 * 40 * 4, dtype=np.float32)
    _check(lib.ref_verify_case(seed, case_index, d, _ptr(xb, C.c_float), _ptr(kb, C.c_float),
                               _ptr(yb, C.c_float)), lib)
    n, k, p, cin, cout = list(d)
    g = geometry(n, k, k, p)
    return dict(n=n, k=k, p=p, cin=cin, cout=cout,
                x=xb[: n * n * cin].reshape(n, n, cin).copy(),
                kernel=kb[: k * k * cin * cout].reshape(k, k, cin, cout).copy(),
                y=yb[: g.out_h * g.out_w * cout].reshape(g.out_h, g.out_w, cout).copy())


def ref_time_fused_batch(mode, x, k, p, workers):
    """Times the reference's segregated CPU path over a batch; returns (out, seconds)."""
    x, k = _f32(x), _f32(k)
    b, n, _, cin = x.shape
    kh, kw, _, cout = k.shape
    g = geometry(n, kh, kw, p)
    out = np.empty((b, g.out_h, g.out_w, cout), dtype=np.float32)
    secs = C.c_double()
    lib = load_ref()
    _check(lib.ref_time_fused_batch_f32(mode, _ptr(x, C.c_float), b, n, cin, _ptr(k, C.c_float),
                                        kh, kw, cout, p, workers, _ptr(out, C.c_float),
                                        C.byref(secs)), lib)
    return out, secs.value


# ------------------------------------------------------------ rounding helpers
def bf16_round(a):
    """Round-to-nearest-even to bfloat16, returned as float32 (for bf16 parity emulation)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def tf32_round(a):
    """Round-to-nearest-even to TF32 (10 explicit mantissa bits), as float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0xFFF + ((u >> 13) & 1)) & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32)

"""Host-side mirror of the reference ``segconv`` operator API over the C ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/segconv, cited per function), operating on torch
tensors in the reference's layouts:

* activations: HWC per image (reference tensor.hpp:57-62), or a batch NHWC;
* kernels: (kh, kw, cin, cout) (tensor.hpp:148-151).

Device tensors are computed in place on the current CUDA stream.  Host (CPU)
tensors are copied to the GPU, computed there and copied back, which is the
value-semantics behaviour of the reference API -- the arithmetic always runs
in the sm_100a kernels; there is no CPU implementation here.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence, Union

import torch

from . import _capi as A

__all__ = [
    "SegconvError", "ShapeError", "ContractError", "StateError", "CudaError", "UnsupportedError",
    "TConvGeometry", "tconv_geometry", "first_active_tap", "active_tap_count",
    "class_input_offset", "sub_kernel_dims", "SubKernelSet", "segregate", "transpose_conv_fused",
    "transpose_conv_fused_parallel", "transpose_conv_naive", "conv2d_valid", "upsample2x_pad",
    "tensors_equal_exact", "tensors_equal_approx", "LayerShape", "OpCounts", "count_ops_naive",
    "count_ops_fused", "select_math", "launch_count", "last_path", "MATHS",
    "transpose_conv_fused_backward", "FusedTConv", "TransposeConvFused", "IoError", "ParseError",
    "TensorFileInfo", "peek_tensor_file", "load_tensor", "save_tensor", "load_tensor_batch",
    "conv2d_valid_backward", "upsample2x_pad_backward", "ConvValid", "Upsample2x",
]


# ------------------------------------------------------------------ errors
class SegconvError(RuntimeError):
    """Base class (reference errors.hpp:10-12)."""


class ShapeError(SegconvError):
    """A dimension constraint was violated (reference errors.hpp:14-18)."""


class ContractError(SegconvError):
    """An API precondition was broken (reference errors.hpp:20-23)."""


class StateError(SegconvError):
    """An operation was called out of order, e.g. backward before forward
    (reference errors.hpp:39, netdemo/layers.hpp:46-48)."""


class IoError(SegconvError):
    """A file could not be opened, read or written (reference errors.hpp:34-37)."""


class ParseError(SegconvError):
    """Malformed file contents; ``byte_offset`` is where parsing stopped
    (reference errors.hpp:25-31)."""

    def __init__(self, msg: str, byte_offset: int = 0):
        super().__init__(msg)
        self.byte_offset = byte_offset


class CudaError(SegconvError):
    """The device could not run the request (no CPU fallback exists)."""


class UnsupportedError(SegconvError):
    """Valid request with no kernel in this build."""


class NcclError(SegconvError):
    """NCCL missing, or a collective of the multi-GPU stack failed."""


_ERR = {A.E_SHAPE: ShapeError, A.E_CONTRACT: ContractError, A.E_CUDA: CudaError,
        A.E_UNSUPPORTED: UnsupportedError, A.E_IO: IoError, A.E_NCCL: NcclError}


def _check(status: int) -> None:
    if status == A.E_PARSE:
        raise ParseError(A.last_error(), int(A.lib().segconv_last_error_offset()))
    if status != A.OK:
        raise _ERR.get(status, SegconvError)(A.last_error())


_DT = {torch.float32: A.F32, torch.float64: A.F64, torch.bfloat16: A.BF16}
_DT_INV = {v: k for k, v in _DT.items()}
MATHS = {"auto": A.MATH_AUTO, "ffma": A.MATH_FFMA, "exact": A.MATH_EXACT, "bf16": A.MATH_BF16,
         "tf32": A.MATH_TF32, "f16x3": A.MATH_F16X3}
_MATH_INV = {v: k for k, v in MATHS.items()}
_ACT = {None: A.EPI_NONE, "none": A.EPI_NONE, "relu": A.EPI_RELU, "tanh": A.EPI_TANH}


def _dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ContractError(f"unsupported dtype {t.dtype} (float32, float64, bfloat16)") from None


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise CudaError("no CUDA device: the segregated transpose convolution runs only on the GPU")
    return torch.device("cuda", torch.cuda.current_device())


def launch_count() -> int:
    """Kernels launched by the C library since it was loaded."""
    return int(A.lib().segconv_launch_count())


# ---------------------------------------------------------------- geometry
@dataclass(frozen=True)
class TConvGeometry:
    """== segconv::TConvGeometry (reference geometry.hpp:18-27)."""
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

    def _c(self) -> A.Geometry:
        return A.Geometry(self.n_in, self.kh, self.kw, self.p_orig, self.p_fused, self.up_h,
                          self.up_w, self.out_h, self.out_w, int(self.trim_extra_row),
                          int(self.trim_extra_col))


def tconv_geometry(n_in: int, kh: int, kw: int, p_orig: int) -> TConvGeometry:
    """reference geometry.hpp:29-53."""
    g = A.Geometry()
    _check(A.lib().segconv_tconv_geometry(int(n_in), int(kh), int(kw), int(p_orig), C.byref(g)))
    return TConvGeometry(g.n_in, g.kh, g.kw, g.p_orig, g.p_fused, g.up_h, g.up_w, g.out_h,
                         g.out_w, bool(g.trim_extra_row), bool(g.trim_extra_col))


def first_active_tap(p: int, r: int) -> int:
    """reference segregation.hpp:24."""
    return A.lib().segconv_first_active_tap(p, r)


def active_tap_count(n: int, p: int, r: int) -> int:
    """reference segregation.hpp:27-30."""
    return A.lib().segconv_active_tap_count(n, p, r)


def class_input_offset(p: int, r: int) -> int:
    """reference segregation.hpp:33-36."""
    return A.lib().segconv_class_input_offset(p, r)


def sub_kernel_dims(n: int):
    """reference segregation.hpp:94-100: the four sub-kernel sizes of an odd n x n kernel."""
    if n < 1:
        raise ContractError("kernel size must be >= 1")
    if n % 2 == 0:
        raise ContractError("sub_kernel_dims is defined for odd sizes only")
    hi, lo = (n + 1) // 2, n // 2
    return [(hi, hi), (hi, lo), (lo, hi), (lo, lo)]


# ------------------------------------------------------------- segregation
class SubKernelSet:
    """Device counterpart of segconv::SubKernelSet<T> (reference segregation.hpp:43-55).

    ``panels`` is one device buffer holding the four parity sub-kernels (class
    r*2+c).  Layout "ref" keeps the reference's (u, v, cin, cout) order (SIMT
    kernels); layout "umma" is the tcgen05 B-operand image (bf16, or fp32
    weights split into fp16 hi + lo planes for math="f16x3").
    """

    def __init__(self, desc: A.SubKernels, panels: torch.Tensor):
        self.desc = desc
        self.panels = panels

    source_kh = property(lambda s: s.desc.source_kh)
    source_kw = property(lambda s: s.desc.source_kw)
    p_orig_parity = property(lambda s: s.desc.p_orig_parity)
    math = property(lambda s: s.desc.math)
    layout = property(lambda s: {A.PANEL_REF: "ref", A.PANEL_KMAJOR: "kmajor",
                                 A.PANEL_UMMA: "umma", A.PANEL_UMMA_FOLD: "fold"}[s.desc.layout])
    dtype = property(lambda s: s.panels.dtype)

    def cin(self) -> int:
        return self.desc.cin

    def cout(self) -> int:
        return self.desc.cout

    def offset(self, r: int, c: int):
        q = r * 2 + c
        return (self.desc.off_r[q], self.desc.off_c[q])

    @property
    def class_input_offsets(self):
        return [self.offset(q >> 1, q & 1) for q in range(4)]

    def sub(self, r: int, c: int) -> torch.Tensor:
        """Class (r, c)'s sub-kernel in the reference (kh, kw, cin, cout) order
        (a view for "ref" panels; a decoded float32 copy for "umma" panels)."""
        d, q = self.desc, r * 2 + c
        kh, kw = d.sub_kh[q], d.sub_kw[q]
        if d.layout == A.PANEL_REF:
            n = kh * kw * d.cin * d.cout_pad
            return self.panels[d.sub_offset[q]: d.sub_offset[q] + n].view(kh, kw, d.cin, d.cout)
        if d.layout == A.PANEL_KMAJOR:
            n = kh * kw * d.cin * d.cout_pad
            flat = self.panels[d.sub_offset[q]: d.sub_offset[q] + n]
            return flat.view(d.cout_pad, kh, kw, d.cin).permute(1, 2, 3, 0)[..., : d.cout]
        planes = 2 if d.dtype == A.F16_SPLIT else 1
        # split-fp16 images hold w * 2^s; the range-guard header after the
        # images stores 2^-s (csrc/tc_guard.cuh)
        inv = self._guard_inv_scale() if d.dtype == A.F16_SPLIT else 1.0
        if d.layout == A.PANEL_UMMA_FOLD:
            # [plane][k_block][chunk][shift*4*cp + q*cp + f][8] over the union window
            CP, KB = d.n_tile, d.k_block
            nkb = (d.cin + KB - 1) // KB
            uc = max(d.off_c[i] + d.sub_kw[i] for i in range(4))
            ur = max(d.off_r[i] + d.sub_kh[i] for i in range(4))
            rows = ur * uc * 4 * CP + (128 - 4 * CP)
            n_img = planes * nkb * (KB // 8) * rows * 8
            blk = self.panels[:n_img].view(planes, nkb, KB // 8, rows, 8).float()
            w = (blk[0] + (blk[1] if planes == 2 else 0)) * inv  # (nkb, CH, rows, 8)
            w = w.permute(2, 0, 1, 3).reshape(rows, nkb * KB)     # (rows, cin_pad)
            out = torch.zeros(kh, kw, d.cin, d.cout, device=w.device)
            for u in range(kh):
                for v in range(kw):
                    s_ = (d.off_r[q] + u) * uc + (d.off_c[q] + v)
                    r0 = s_ * 4 * CP + q * CP
                    out[u, v] = w[r0: r0 + d.cout, : d.cin].t()
            return out
        # UMMA image: blocks (n_tile, k_block, tap) x [plane][chunk][row][8]
        NT, KB = d.n_tile, d.k_block
        nkb = (d.cin + KB - 1) // KB
        ntl = d.cout_pad // NT
        taps = sum(d.sub_kh[i] * d.sub_kw[i] for i in range(4))
        n_img = ntl * nkb * taps * planes * (KB // 8) * NT * 8
        blk = self.panels[:n_img].view(ntl, nkb, taps, planes, KB // 8, NT, 8).float()
        w = (blk[:, :, :, 0] + (blk[:, :, :, 1] if planes == 2 else 0)) * inv
        # -> (tap, kb, chunk, e, nt, n) -> (tap, cin_pad, cout_pad)
        w = w.permute(2, 1, 3, 5, 0, 4).reshape(taps, nkb * KB, ntl * NT)
        t0 = int(d.sub_offset[q])
        return w[t0: t0 + kh * kw, : d.cin, : d.cout].reshape(kh, kw, d.cin, d.cout)

    def _guard_inv_scale(self) -> float:
        d = self.desc
        if d.layout not in (A.PANEL_UMMA_FOLD, A.PANEL_UMMA):
            return 1.0
        off = d.total_elems - (16 + d.source_kh * d.source_kw * d.cin * d.cout * 4) // 2
        return float(self.panels[off: off + 2].view(torch.float32)[0])

    @property
    def subs(self):
        return [self.sub(q >> 1, q & 1) for q in range(4)]


def last_path() -> str:
    """Kernel family the last transpose_conv_fused call on this thread ran."""
    return (A.lib().segconv_last_path() or b"").decode()


def select_math(x_dtype: torch.dtype, panel_dtype: torch.dtype, cin: int, cout: int, kh: int,
                kw: int) -> str:
    """What math="auto" resolves to for a problem."""
    m = A.lib().segconv_select_math(_DT[x_dtype], _DT[panel_dtype], cin, cout, kh, kw)
    return _MATH_INV[m]


_PANEL_TORCH = {A.F32: torch.float32, A.F64: torch.float64, A.BF16: torch.bfloat16,
                A.F16_SPLIT: torch.float16}


def segregate(kernel: torch.Tensor, p_orig: int, *, math: str = "auto",
              x_dtype: Optional[torch.dtype] = None) -> SubKernelSet:
    """reference segregation.hpp:61-89: split a (kh, kw, cin, cout) kernel into
    the four parity panels, on the device.  ``math`` selects the consumer
    ("ffma"/"exact" -> reference-layout panels; "bf16"/"f16x3" -> tcgen05
    panel image; "auto" decides from the activation dtype (default: the
    kernel's dtype) and the shape)."""
    if kernel.dim() != 4:
        raise ShapeError(f"kernel must be (kh, kw, cin, cout), got {tuple(kernel.shape)}")
    kh, kw, cin, cout = (int(v) for v in kernel.shape)
    if kh < 1 or kw < 1:
        raise ContractError("cannot segregate a spatially empty kernel")
    if p_orig < 0:
        raise ContractError("padding must be non-negative")
    if math not in MATHS:
        raise ContractError(f"unknown math {math!r}")
    dev = _device()
    k = kernel.to(dev).contiguous()
    kd = _dtype_code(k)
    xd = _DT[x_dtype] if x_dtype is not None else kd
    desc = A.SubKernels()
    _check(A.lib().segconv_subkernels_for_math(kh, kw, cin, cout, int(p_orig), xd, MATHS[math],
                                               C.byref(desc)))
    if desc.layout == A.PANEL_REF and desc.dtype != kd:
        k = k.to(_PANEL_TORCH[desc.dtype])
        kd = desc.dtype
    panels = torch.empty(max(1, desc.total_elems), dtype=_PANEL_TORCH[desc.dtype], device=dev)
    _check(A.lib().segconv_segregate(k.data_ptr(), kd, C.byref(desc), panels.data_ptr(),
                                     _stream()))
    return SubKernelSet(desc, panels)


# ------------------------------------------------------------ fused (hot)
def _as_batch(x: torch.Tensor):
    if x.dim() == 3:
        return x.unsqueeze(0), True
    if x.dim() == 4:
        return x, False
    raise ShapeError(f"input must be HWC or NHWC, got {tuple(x.shape)}")


def _epilogue(bias, activation):
    if activation not in _ACT:
        raise ContractError(f"unknown activation {activation!r} (relu, tanh, None)")
    epi = _ACT[activation]
    if bias is not None:
        epi |= A.EPI_BIAS
    return epi


def transpose_conv_fused(x: torch.Tensor, k: Union[SubKernelSet, torch.Tensor],
                         geom: Union[TConvGeometry, int, None] = None, *,
                         bias: Optional[torch.Tensor] = None, activation: Optional[str] = None,
                         math: Optional[str] = None, out_dtype: Optional[torch.dtype] = None,
                         out: Optional[torch.Tensor] = None, staging=None,
                         chunks: Optional[int] = None, sync: bool = True) -> torch.Tensor:
    """Segregated 2x transpose convolution.

    ``transpose_conv_fused(x, sks, geom)``  -- reference fused_tconv.hpp:69-82
    ``transpose_conv_fused(x, kernel, p)``  -- reference fused_tconv.hpp:85-92

    ``x`` is (N, N, cin) or (B, N, N, cin); the result is (out_h, out_w, cout)
    or (B, out_h, out_w, cout).  Optional fused epilogue: ``bias`` (cout,) then
    ``activation`` "relu" | "tanh".

    A host (CPU) ``x`` gives a host result, as the reference's value-semantics
    call does, through segconv_transpose_conv_fused_host: batch slices are
    uploaded, computed and downloaded in a pipeline (``chunks`` slices; use
    page-locked ``x`` / ``out`` for overlap).  ``staging`` = (device x, device y)
    buffers to reuse; ``sync=False`` leaves the result pending on the current
    stream.
    """
    xb, squeeze = _as_batch(x)
    if isinstance(k, torch.Tensor):
        p = int(geom if geom is not None else 0)
        if k.dim() != 4:
            raise ShapeError("kernel must be (kh, kw, cin, cout)")
        g = tconv_geometry(xb.shape[1], int(k.shape[0]), int(k.shape[1]), p)
        if xb.shape[1] != xb.shape[2]:
            raise ContractError(f"transpose conv expects a square input, got "
                                f"{xb.shape[1]}x{xb.shape[2]}")
        sks = segregate(k, p, math=math or "auto", x_dtype=xb.dtype)
        math = None
    else:
        if not isinstance(geom, TConvGeometry):
            raise ContractError("transpose_conv_fused(x, sks, geom) needs a TConvGeometry")
        sks, g = k, geom
        if xb.shape[1] != g.n_in or xb.shape[2] != g.n_in:
            raise ContractError(f"input is {xb.shape[1]}x{xb.shape[2]} but geometry was built "
                                f"for {g.n_in}x{g.n_in}")
    m = MATHS[math] if math is not None else A.MATH_AUTO
    host = not xb.is_cuda
    if host:
        y = _fused_host(xb, sks, g, m, bias, activation, out_dtype, out, staging, chunks, sync)
        return y[0] if squeeze else y
    dev = _device()
    xd = xb.to(dev).contiguous()
    b, cin = int(xd.shape[0]), int(xd.shape[3])
    odt = out_dtype or xd.dtype
    if out is None:
        y = torch.empty((b, g.out_h, g.out_w, sks.cout()), dtype=odt, device=dev)
    else:
        y = out if out.dim() == 4 else out.unsqueeze(0)
        if tuple(y.shape) != (b, g.out_h, g.out_w, sks.cout()) or not y.is_contiguous():
            raise ContractError("`out` has the wrong shape or is not contiguous")
    epi = _epilogue(bias, activation)
    bptr = None
    if bias is not None:
        bias = bias.to(dev, torch.float32).contiguous()
        if bias.numel() != sks.cout():
            raise ContractError(f"bias has {bias.numel()} elements, cout is {sks.cout()}")
        bptr = bias.data_ptr()
    gc = g._c()
    _check(A.lib().segconv_transpose_conv_fused(
        xd.data_ptr(), _dtype_code(xd), b, int(xd.shape[1]), cin, C.byref(sks.desc),
        sks.panels.data_ptr(), C.byref(gc), bptr, epi, m, y.data_ptr(), _dtype_code(y),
        _stream()))
    if host:
        y = y.cpu()
    return y[0] if squeeze else y


def transpose_conv_fused_backward(x: torch.Tensor, kernel: torch.Tensor, p_orig: int,
                                  grad_out: torch.Tensor, *, math: Optional[str] = None,
                                  input_grad: bool = True, kernel_grad: bool = True,
                                  grad_kernel: Optional[torch.Tensor] = None,
                                  grad_input: Optional[torch.Tensor] = None):
    """Gradients of the fused layer -- reference netdemo/layers.hpp:171-211
    (net::FusedTConv::backward), batched.

    ``x`` (B, N, N, cin) or (N, N, cin) is the forward input, ``kernel`` the
    original (kh, kw, cin, cout) kernel, ``grad_out`` the output gradient.
    Returns ``(grad_input, grad_kernel)`` (either None when not requested);
    grad_input has x's dtype, grad_kernel is float32 (float64 for double data)
    and summed over the batch.  Passing ``grad_kernel`` accumulates into it, as
    the reference's grad_ does across backward calls; ``grad_input`` (a
    contiguous CUDA tensor of x's batched shape and dtype) receives the input
    gradient in place.  ``math``: "exact"
    (bit-identical to the reference, float/double), "ffma", "bf16", "f16x3"
    (fp32: the input gradient on the tensor cores in split-fp16 math where the
    shape allows -- 2 cout a multiple of 64, cin >= 64 -- the kernel gradient,
    whose pixel sums are far longer than the tensor cores' accumulation bound,
    on FFMA; a device-side range guard hands extreme dynamic ranges to FFMA),
    None (auto: bf16 for bf16 data, f16x3 for float32, ffma for float64).
    """
    xb, squeeze = _as_batch(x)
    gb, _ = _as_batch(grad_out)
    if kernel.dim() != 4:
        raise ShapeError(f"kernel must be (kh, kw, cin, cout), got {tuple(kernel.shape)}")
    kh, kw, kcin, cout = (int(v) for v in kernel.shape)
    b, n, n2, cin = (int(v) for v in xb.shape)
    if n != n2:
        raise ContractError(f"fused_tconv expects a square input, got {n}x{n2}")
    if kcin != cin:
        raise ContractError(f"channel mismatch: input has {cin}, kernel expects {kcin}")
    g = tconv_geometry(n, kh, kw, int(p_orig))
    if tuple(gb.shape) != (b, g.out_h, g.out_w, cout):
        raise ContractError("fused_tconv: output gradient shape mismatch")
    if math is not None and math not in MATHS:
        raise ContractError(f"unknown math {math!r}")
    dev = _device()
    dt = xb.dtype
    xd = xb.to(dev).contiguous()
    gd = gb.to(dev, dt).contiguous()
    kd = kernel.to(dev, dt).contiguous()
    if input_grad and grad_input is not None:
        if tuple(grad_input.shape) != tuple(xd.shape) or grad_input.dtype != dt or \
                not grad_input.is_cuda or not grad_input.is_contiguous():
            raise ContractError("grad_input must be a contiguous CUDA tensor of the input's shape and dtype")
        gx = grad_input
    else:
        gx = torch.empty_like(xd) if input_grad else None
    acc_dt = torch.float64 if dt == torch.float64 else torch.float32
    acc = 0
    if kernel_grad:
        if grad_kernel is not None:
            if tuple(grad_kernel.shape) != (kh, kw, cin, cout) or grad_kernel.dtype != acc_dt or \
                    not grad_kernel.is_cuda or not grad_kernel.is_contiguous():
                raise ContractError(f"grad_kernel must be a contiguous {acc_dt} CUDA tensor of the "
                                    "kernel's shape")
            gk, acc = grad_kernel, 1
        else:
            gk = torch.empty((kh, kw, cin, cout), dtype=acc_dt, device=dev)
    else:
        gk = None
    m = MATHS[math] if math is not None else A.MATH_AUTO
    _check(A.lib().segconv_transpose_conv_fused_backward(
        xd.data_ptr(), gd.data_ptr(), _dtype_code(xd), b, n, cin, kd.data_ptr(), kh, kw, cout,
        int(p_orig), m, gx.data_ptr() if gx is not None else None,
        gk.data_ptr() if gk is not None else None, acc, _stream()))
    if gx is not None and squeeze:
        gx = gx[0]
    return gx, gk


class FusedTConv:
    """Trainable fused 2x transpose convolution -- the reference's
    net::FusedTConv<T> (netdemo/layers.hpp:150-230) on the GPU, batched.

    forward(x) caches the input and runs the segregated kernels; backward(g)
    returns the input gradient and adds the kernel gradient into ``grad``;
    params() exposes (values, grads); on_params_updated() re-segregates."""

    def __init__(self, kernel: torch.Tensor, p: int, *, math: Optional[str] = None):
        self.kernel_ = kernel.to(_device()).contiguous()
        self.p_ = int(p)
        self.math = math
        acc_dt = torch.float64 if self.kernel_.dtype == torch.float64 else torch.float32
        self.grad = torch.zeros(self.kernel_.shape, dtype=acc_dt, device=self.kernel_.device)
        self._input = None
        self.on_params_updated()

    def name(self) -> str:
        return "fused_tconv"

    def kernel(self) -> torch.Tensor:
        return self.kernel_

    def padding(self) -> int:
        return self.p_

    def on_params_updated(self) -> None:
        self.sks_ = segregate(self.kernel_, self.p_, math=self.math or "auto")

    def params(self):
        return [(self.kernel_, self.grad)]

    def zero_grads(self) -> None:
        self.grad.zero_()

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        xb, _ = _as_batch(x)
        if xb.shape[1] != xb.shape[2]:
            raise ContractError(f"fused_tconv expects a square input, got "
                                f"{xb.shape[1]}x{xb.shape[2]}")
        self.geom_ = tconv_geometry(int(xb.shape[1]), int(self.kernel_.shape[0]),
                                    int(self.kernel_.shape[1]), self.p_)
        self._input = x.to(_device()).contiguous()
        return transpose_conv_fused(self._input, self.sks_, self.geom_,
                                    math=self.math if self.math != "auto" else None)

    def backward(self, g: torch.Tensor) -> torch.Tensor:
        if self._input is None:
            raise StateError("fused_tconv: backward called before forward")
        gx, _ = transpose_conv_fused_backward(self._input, self.kernel_, self.p_, g,
                                              math=self._bwd_math(), grad_kernel=self.grad)
        return gx

    def _bwd_math(self):
        if self.math in (None, "auto"):
            return None
        return "bf16" if self.math in ("bf16",) else ("exact" if self.math == "exact" else "ffma")


class ConvValid:
    """Trainable valid correlation -- the reference's net::ConvValid<T>
    (netdemo/layers.hpp:84-137) on the GPU, batched; same conventions as
    FusedTConv."""

    def __init__(self, kernel: torch.Tensor, *, math: Optional[str] = None):
        self.kernel_ = kernel.to(_device()).contiguous()
        self.math = math
        acc_dt = torch.float64 if self.kernel_.dtype == torch.float64 else torch.float32
        self.grad = torch.zeros(self.kernel_.shape, dtype=acc_dt, device=self.kernel_.device)
        self._input = None

    def name(self) -> str:
        return "conv_valid"

    def kernel(self) -> torch.Tensor:
        return self.kernel_

    def params(self):
        return [(self.kernel_, self.grad)]

    def zero_grads(self) -> None:
        self.grad.zero_()

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        self._input = x.to(_device()).contiguous()
        return conv2d_valid(self._input, self.kernel_)

    def backward(self, g: torch.Tensor) -> torch.Tensor:
        if self._input is None:
            raise StateError("conv_valid: backward called before forward")
        gx, _ = conv2d_valid_backward(self._input, self.kernel_, g, math=self.math,
                                      grad_kernel=self.grad)
        return gx


class Upsample2x:
    """The reference's net::Upsample2x<T> (netdemo/layers.hpp:54-79) with the
    conventional path's padding p folded in (pad(upsample2x(x), p))."""

    def __init__(self, p: int = 0):
        self.p = int(p)
        self._n = None

    def name(self) -> str:
        return "upsample2x"

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        self._n = int(x.shape[-2])
        return upsample2x_pad(x, self.p)

    def backward(self, g: torch.Tensor) -> torch.Tensor:
        if self._n is None:
            raise StateError("upsample2x: backward called before forward")
        return upsample2x_pad_backward(g, self._n, self.p)


class TransposeConvFused(torch.autograd.Function):
    """torch.autograd wrapper: y = transpose_conv_fused(x, kernel, p) with the
    backward of transpose_conv_fused_backward (NHWC tensors, kernel (kh, kw,
    cin, cout))."""

    @staticmethod
    def forward(ctx, x, kernel, p):
        ctx.save_for_backward(x, kernel)
        ctx.p = int(p)
        return transpose_conv_fused(x, kernel, int(p))

    @staticmethod
    def backward(ctx, grad_out):
        x, kernel = ctx.saved_tensors
        gx, gk = transpose_conv_fused_backward(
            x, kernel, ctx.p, grad_out.contiguous(), input_grad=ctx.needs_input_grad[0],
            kernel_grad=ctx.needs_input_grad[1])
        if gk is not None:
            gk = gk.to(kernel.dtype)
        return gx, gk, None


# ------------------------------------------------------------ SGC1 files
@dataclass(frozen=True)
class TensorFileInfo:
    """== segconv::TensorFileInfo (reference tensor_io.hpp:48-51)."""
    height: int
    width: int
    channels: int
    precision: str  # "f32" | "f64"


_PREC = {0: "f32", 1: "f64"}
_PREC_T = {"f32": torch.float32, "f64": torch.float64}


def peek_tensor_file(path: str) -> TensorFileInfo:
    """reference tensor_io.hpp:53-74: parse the 20-byte SGC1 header."""
    info = A.TensorFileInfo()
    _check(A.lib().segconv_peek_tensor_file(os.fsencode(path), C.byref(info)))
    return TensorFileInfo(info.height, info.width, info.channels, _PREC[info.precision])


def load_tensor(path: str, dtype: Optional[torch.dtype] = None, *, device=None) -> torch.Tensor:
    """reference tensor_io.hpp:76-91 (load_tensor<T>): an (h, w, c) tensor.
    ``dtype`` (float32/float64) must match the stored precision
    (ContractError); default: the stored one.  ``device`` moves the result."""
    info = peek_tensor_file(path)
    dt = dtype or _PREC_T[info.precision]
    if dt not in (torch.float32, torch.float64):
        raise ContractError("SGC1 stores float32 or float64 tensors")
    pin = device is not None and torch.device(device).type == "cuda" and torch.cuda.is_available()
    t = torch.empty((info.height, info.width, info.channels), dtype=dt, pin_memory=pin)
    _check(A.lib().segconv_load_tensor(os.fsencode(path), _DT[dt], t.data_ptr(),
                                       t.numel() * t.element_size()))
    return t.to(device, non_blocking=True) if device is not None else t


def save_tensor(t: torch.Tensor, path: str) -> None:
    """reference tensor_io.hpp:93-103 (save_tensor<T>): t is (h, w, c) float32/float64."""
    if t.dim() != 3:
        raise ShapeError(f"SGC1 holds (h, w, c) tensors, got {tuple(t.shape)}")
    if t.dtype not in (torch.float32, torch.float64):
        raise ContractError("SGC1 stores float32 or float64 tensors")
    h = t.detach().cpu().contiguous()
    _check(A.lib().segconv_save_tensor(os.fsencode(path), h.data_ptr() if h.numel() else None,
                                       int(h.shape[0]), int(h.shape[1]), int(h.shape[2]),
                                       _DT[h.dtype]))


def load_tensor_batch(paths, dtype: Optional[torch.dtype] = None, *, device=None) -> torch.Tensor:
    """Many SGC1 files of one shape -> a (B, h, w, c) batch.  With a CUDA
    ``device`` the files are read into a page-locked staging buffer and each
    image's upload is queued as soon as it is read (reads overlap copies)."""
    paths = list(paths)
    if not paths:
        raise ContractError("empty batch")
    info = peek_tensor_file(paths[0])
    dt = dtype or _PREC_T[info.precision]
    shape = (len(paths), info.height, info.width, info.channels)
    cuda = device is not None and torch.device(device).type == "cuda"
    host = torch.empty(shape, dtype=dt, pin_memory=cuda)
    dev = torch.empty(shape, dtype=dt, device=device) if cuda else None
    arr = (C.c_char_p * len(paths))(*[os.fsencode(p) for p in paths])
    _check(A.lib().segconv_load_tensor_batch(arr, len(paths), _DT[dt], host.data_ptr(),
                                             dev.data_ptr() if dev is not None else None,
                                             _stream() if cuda else None))
    if cuda:
        torch.cuda.current_stream().synchronize()  # the staging buffer is released on return
        return dev
    return host if device is None else host.to(device)


def _fused_host(xb, sks, g, m, bias, activation, out_dtype, out, staging, chunks, sync):
    """Host-buffer call: C ABI segconv_transpose_conv_fused_host (pipelined copies)."""
    dev = _device()
    xh = xb.contiguous()
    b, cin = int(xh.shape[0]), int(xh.shape[3])
    odt = out_dtype or xh.dtype
    shape = (b, g.out_h, g.out_w, sks.cout())
    if out is None:
        yh = torch.empty(shape, dtype=odt, pin_memory=torch.cuda.is_available())
    else:
        yh = out if out.dim() == 4 else out.unsqueeze(0)
        if tuple(yh.shape) != shape or not yh.is_contiguous() or yh.is_cuda:
            raise ContractError("`out` must be a contiguous host tensor of the output shape")
    if staging is None:
        xd = torch.empty(xh.shape, dtype=xh.dtype, device=dev)
        yd = torch.empty(shape, dtype=yh.dtype, device=dev)
    else:
        xd, yd = staging
        if tuple(xd.shape) != tuple(xh.shape) or tuple(yd.shape) != shape or \
                xd.dtype != xh.dtype or yd.dtype != yh.dtype:
            raise ContractError("staging buffers do not match the input / output")
    epi = _epilogue(bias, activation)
    bptr = None
    if bias is not None:
        bias = bias.to(dev, torch.float32).contiguous()
        if bias.numel() != sks.cout():
            raise ContractError(f"bias has {bias.numel()} elements, cout is {sks.cout()}")
        bptr = bias.data_ptr()
    gc = g._c()
    _check(A.lib().segconv_transpose_conv_fused_host(
        xh.data_ptr(), xd.data_ptr(), _dtype_code(xh), b, int(xh.shape[1]), cin,
        C.byref(sks.desc), sks.panels.data_ptr(), C.byref(gc), bptr, epi, m, yd.data_ptr(),
        yh.data_ptr(), _dtype_code(yh), int(chunks or 0), _stream()))
    if sync:
        torch.cuda.current_stream().synchronize()
    return yh


def transpose_conv_fused_parallel(x: torch.Tensor, sks: SubKernelSet, geom: TConvGeometry,
                                  workers: int, **kw) -> torch.Tensor:
    """reference fused_tconv.hpp:101-147.  The reference splits cout across CPU
    threads; here the GPU grid is the parallelism, so ``workers`` is validated
    (ContractError if < 1, fused_tconv.hpp:104) and otherwise has no effect --
    the result equals transpose_conv_fused exactly, as in the reference."""
    if workers < 1:
        raise ContractError("worker count must be >= 1")
    return transpose_conv_fused(x, sks, geom, **kw)


# ------------------------------------------------------- conventional path
def upsample2x_pad(x: torch.Tensor, p: int) -> torch.Tensor:
    """reference tensor.hpp:224-259: pad(upsample2x(x), p) on the device."""
    xb, squeeze = _as_batch(x)
    dev = _device()
    host = not xb.is_cuda
    xd = xb.to(dev).contiguous()
    b, h, w, c = (int(v) for v in xd.shape)
    if h != w:
        raise ContractError("upsample2x_pad expects square maps")
    U = 2 * h - 1 + 2 * p
    up = torch.empty((b, U, U, c), dtype=xd.dtype, device=dev)
    _check(A.lib().segconv_upsample2x_pad(xd.data_ptr(), _dtype_code(xd), b, h, c, int(p),
                                          up.data_ptr(), _stream()))
    if host:
        up = up.cpu()
    return up[0] if squeeze else up


def upsample2x_pad_backward(grad_up: torch.Tensor, n_in: int, p: int) -> torch.Tensor:
    """Gradient of upsample2x_pad (reference netdemo/layers.hpp:66-73 after the pad
    crop): the (B, up, up, c) gradient sampled at (2i + p, 2j + p)."""
    gb, squeeze = _as_batch(grad_up)
    dev = _device()
    gd = gb.to(dev).contiguous()
    b, U, U2, c = (int(v) for v in gd.shape)
    if U != U2 or U != 2 * int(n_in) - 1 + 2 * int(p):
        raise ContractError(f"upsampled gradient is {U}x{U2}, expected {2 * n_in - 1 + 2 * p}")
    gx = torch.empty((b, int(n_in), int(n_in), c), dtype=gd.dtype, device=dev)
    _check(A.lib().segconv_upsample2x_pad_backward(gd.data_ptr(), _dtype_code(gd), b, int(n_in), c,
                                                   int(p), gx.data_ptr(), _stream()))
    return gx[0] if squeeze else gx


def conv2d_valid(src: torch.Tensor, k: torch.Tensor, *, bias=None, activation=None,
                 math: Optional[str] = None) -> torch.Tensor:
    """reference reference_ops.hpp:86-108.  ``math="exact"`` (float/double):
    the reference's accumulation order, bit-identical to its CPU result."""
    sb, squeeze = _as_batch(src)
    dev = _device()
    host = not sb.is_cuda
    sd = sb.to(dev).contiguous()
    kd = k.to(dev, sd.dtype).contiguous()
    if kd.dim() != 4:
        raise ShapeError("kernel must be (kh, kw, cin, cout)")
    kh, kw, kc, cout = (int(v) for v in kd.shape)
    b, h, w, cin = (int(v) for v in sd.shape)
    if kh < 1 or kw < 1:
        raise ShapeError("conv2d_valid needs a non-empty kernel")
    if kc != cin:
        raise ContractError(f"channel mismatch: input has {cin}, kernel expects {kc}")
    oh, ow = h - kh + 1, w - kw + 1
    if oh < 1 or ow < 1:
        raise ShapeError(f"kernel {kh}x{kw} does not fit input {h}x{w}")
    y = torch.empty((b, oh, ow, cout), dtype=sd.dtype, device=dev)
    epi = _epilogue(bias, activation)
    bptr = bias.to(dev, torch.float32).contiguous().data_ptr() if bias is not None else None
    _check(A.lib().segconv_conv2d_valid(sd.data_ptr(), _dtype_code(sd), b, h, w, cin,
                                        kd.data_ptr(), kh, kw, cout, bptr, epi,
                                        MATHS[math or "auto"], y.data_ptr(), _stream()))
    if host:
        y = y.cpu()
    return y[0] if squeeze else y


def conv2d_valid_backward(src: torch.Tensor, kernel: torch.Tensor, grad_out: torch.Tensor, *,
                          math: Optional[str] = None, input_grad: bool = True,
                          kernel_grad: bool = True, grad_kernel: Optional[torch.Tensor] = None):
    """Gradients of conv2d_valid -- reference netdemo/layers.hpp:98-122
    (net::ConvValid::backward), batched; same conventions as
    transpose_conv_fused_backward."""
    sb, squeeze = _as_batch(src)
    gb, _ = _as_batch(grad_out)
    if kernel.dim() != 4:
        raise ShapeError(f"kernel must be (kh, kw, cin, cout), got {tuple(kernel.shape)}")
    kh, kw, kcin, cout = (int(v) for v in kernel.shape)
    b, h, w, cin = (int(v) for v in sb.shape)
    if kcin != cin:
        raise ContractError(f"channel mismatch: input has {cin}, kernel expects {kcin}")
    oh, ow = h - kh + 1, w - kw + 1
    if oh < 1 or ow < 1:
        raise ShapeError(f"kernel {kh}x{kw} does not fit input {h}x{w}")
    if tuple(gb.shape) != (b, oh, ow, cout):
        raise ContractError("conv_valid: output gradient shape mismatch")
    if math is not None and math not in MATHS:
        raise ContractError(f"unknown math {math!r}")
    dev = _device()
    dt = sb.dtype
    sd, gd, kd = sb.to(dev).contiguous(), gb.to(dev, dt).contiguous(), kernel.to(dev, dt).contiguous()
    gx = torch.empty_like(sd) if input_grad else None
    acc_dt = torch.float64 if dt == torch.float64 else torch.float32
    acc = 0
    gk = None
    if kernel_grad:
        if grad_kernel is not None:
            if tuple(grad_kernel.shape) != (kh, kw, cin, cout) or grad_kernel.dtype != acc_dt or \
                    not grad_kernel.is_cuda or not grad_kernel.is_contiguous():
                raise ContractError(f"grad_kernel must be a contiguous {acc_dt} CUDA tensor of the "
                                    "kernel's shape")
            gk, acc = grad_kernel, 1
        else:
            gk = torch.empty((kh, kw, cin, cout), dtype=acc_dt, device=dev)
    m = MATHS[math] if math is not None else A.MATH_AUTO
    _check(A.lib().segconv_conv2d_valid_backward(
        sd.data_ptr(), gd.data_ptr(), _dtype_code(sd), b, h, w, cin, kd.data_ptr(), kh, kw, cout, m,
        gx.data_ptr() if gx is not None else None, gk.data_ptr() if gk is not None else None, acc,
        _stream()))
    if gx is not None and squeeze:
        gx = gx[0]
    return gx, gk


def transpose_conv_naive(x: torch.Tensor, k: torch.Tensor, p: int, *, bias=None,
                         activation=None, workspace: Optional[torch.Tensor] = None,
                         math: Optional[str] = None) -> torch.Tensor:
    """reference reference_ops.hpp:116-133: upsample, pad, valid-correlate
    (the conventional baseline; materialises the (2N-1+2p)^2 map).
    ``math="exact"``: bit-identical to the reference (and to the fused op's
    EXACT mode, the reference's fused == naive guarantee)."""
    xb, squeeze = _as_batch(x)
    dev = _device()
    host = not xb.is_cuda
    xd = xb.to(dev).contiguous()
    if k.dim() != 4:
        raise ShapeError("kernel must be (kh, kw, cin, cout)")
    kd = k.to(dev, xd.dtype).contiguous()
    kh, kw, kc, cout = (int(v) for v in kd.shape)
    b, h, w, cin = (int(v) for v in xd.shape)
    if kc != cin:
        raise ContractError(f"channel mismatch: input has {cin}, kernel expects {kc}")
    g = tconv_geometry(h, kh, kw, p)
    if h != w:
        raise ContractError(f"transpose conv expects a square input, got {h}x{w}")
    need = int(A.lib().segconv_naive_workspace_bytes(_dtype_code(xd), b, h, cin, int(p)))
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)
    y = torch.empty((b, g.out_h, g.out_w, cout), dtype=xd.dtype, device=dev)
    epi = _epilogue(bias, activation)
    bptr = bias.to(dev, torch.float32).contiguous().data_ptr() if bias is not None else None
    _check(A.lib().segconv_transpose_conv_naive(
        xd.data_ptr(), _dtype_code(xd), b, h, cin, kd.data_ptr(), kh, kw, cout, int(p),
        workspace.data_ptr(), workspace.numel() * workspace.element_size(), bptr, epi,
        MATHS[math or "auto"], y.data_ptr(), _stream()))
    if host:
        y = y.cpu()
    return y[0] if squeeze else y


# ------------------------------------------------------------ comparators
def tensors_equal_exact(a: torch.Tensor, b: torch.Tensor) -> bool:
    """reference tensor.hpp:263-272: same shape and IEEE-equal (+0 == -0)."""
    return tuple(a.shape) == tuple(b.shape) and bool(torch.equal(a.cpu(), b.cpu()) or
                                                     bool((a.cpu() == b.cpu()).all()))


def tensors_equal_approx(a: torch.Tensor, b: torch.Tensor, rel_tol: float) -> bool:
    """reference tensor.hpp:275-286: |a-b| <= tol * max(|a|, |b|, 1)."""
    if tuple(a.shape) != tuple(b.shape):
        return False
    a64, b64 = a.detach().double().cpu(), b.detach().double().cpu()
    scale = torch.maximum(torch.maximum(a64.abs(), b64.abs()), torch.ones_like(a64))
    return bool(((a64 - b64).abs() <= rel_tol * scale).all())


# ---------------------------------------------------------------- counts
@dataclass(frozen=True)
class LayerShape:
    """reference analysis.hpp:15-22."""
    n_in: int
    cin: int
    cout: int
    kh: int
    kw: int
    p_orig: int


@dataclass(frozen=True)
class OpCounts:
    mults: int
    adds: int


def _counts(s: LayerShape):
    o = (C.c_uint64 * 4)()
    _check(A.lib().segconv_count_ops(s.n_in, s.cin, s.cout, s.kh, s.kw, s.p_orig, o))
    return [int(v) for v in o]


def count_ops_naive(s: LayerShape) -> OpCounts:
    """reference analysis.hpp:31-41."""
    v = _counts(s)
    return OpCounts(v[0], v[1])


def count_ops_fused(s: LayerShape) -> OpCounts:
    """reference analysis.hpp:48-67 (useful MACs: the metric numerator)."""
    v = _counts(s)
    return OpCounts(v[2], v[3])

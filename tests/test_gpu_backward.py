"""GPU parity of the backward pass of the fused layer (reference
netdemo/layers.hpp:171-211, net::FusedTConv::backward) against the C oracle,
which tests/test_oracle.py pins bit-exactly to the reference.

Bars: EXACT math is bit-identical to the reference (golden vectors, float and
double); FFMA is within the fp32 rounding bound 1e-5 * sum|terms| of the oracle
(summation-order differences only) and bit-exact on integer data; the bf16 tensor-core input
gradient equals the oracle's fp32 result rounded to bf16 on integer data and is
within 1e-2 (the bf16 output rounding) on real data.
"""
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2209_03704_b200 import segconv as sc

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")


def scaled_err(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape
    if got.size == 0:
        return 0.0
    return float((np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), 1.0)).max())


def gpu_bwd(x, k, p, gy, math=None, dtype=None, **kw):
    dt = dtype or {np.float32: torch.float32, np.float64: torch.float64}[x.dtype.type]
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(dt)  # noqa: E731
    gx, gk = sc.transpose_conv_fused_backward(t(x), t(k), p, t(gy), math=math, **kw)
    torch.cuda.synchronize()
    return (None if gx is None else gx.double().cpu().numpy(),
            None if gk is None else gk.double().cpu().numpy(), sc.last_path())


def test_exact_matches_reference_goldens_bit_for_bit():
    z = np.load(os.path.join(G, "backward.npz"))
    for i in range(int(z["count"])):
        dims = [int(v) for v in z[f"b{i}_dims"]]
        x, k, gy = z[f"b{i}_x"], z[f"b{i}_k"], z[f"b{i}_gy"]
        gx, gk, path = gpu_bwd(x, k, dims[6], gy, math="exact")
        assert path == "bwd:simt-exact+simt-exact"
        np.testing.assert_array_equal(gx.astype(x.dtype), z[f"b{i}_gx"], err_msg=f"case {i} {dims}")
        np.testing.assert_array_equal(gk.astype(x.dtype), z[f"b{i}_gk"], err_msg=f"case {i} {dims}")


@pytest.mark.parametrize("b,n,cin,cout,k,p", [
    (2, 16, 64, 32, 3, 0),    # C2 layer shape (reduced batch)
    (3, 8, 48, 20, 4, 2),     # partial channel tiles, p_fused = 1
    (1, 5, 3, 7, 5, 3),       # tiny channels, odd p
    (2, 9, 130, 70, 3, 1),    # channel tiles past 128
    (4, 6, 16, 8, 1, 0),      # 1x1 kernel: classes without taps
    (2, 11, 128, 3, 3, 0),    # C5 layer d shape (fp32)
    (1, 64, 64, 3, 5, 0),     # C4 family (narrow-output kernels), reduced size
    (2, 20, 40, 1, 4, 2),     # narrow: partial channel block, one feature
    (1, 130, 16, 4, 3, 1),    # narrow: rows wider than one 128-pixel segment
    (1, 64, 10, 2, 3, 1),     # narrow: channels not a multiple of 4 (scalar loads / stores)
    (2, 64, 72, 3, 4, 2),     # narrow: two channel blocks, p_fused = 1, two images
])
def test_ffma_f32(b, n, cin, cout, k, p):
    rng = np.random.default_rng(b * 1000 + n * 10 + k)
    x = rng.uniform(-1, 1, (b, n, n, cin)).astype(np.float32)
    kk = (rng.standard_normal((k, k, cin, cout)) * 0.05).astype(np.float32)
    g = oracle.geometry(n, k, k, p)
    gy = rng.uniform(-1, 1, (b, g.out_h, g.out_w, cout)).astype(np.float32)
    wx, wk = oracle.tconv_backward(x, kk, p, gy)
    gx, gk, path = gpu_bwd(x, kk, p, gy, math="ffma")
    kind = "simt-narrow" if cout <= 4 and n >= 64 and k * k * cout <= 80 else "simt-ffma"
    assert path == f"bwd:{kind}+{kind}"
    # summation order differs (tiles, pixel splits): bar = fp32 rounding bound
    # 1e-5 * sum|terms| per element (the kernel gradient sums up to 2 * 16 * 16
    # pixels with cancellation)
    ax, ak = oracle.tconv_backward(np.abs(x), np.abs(kk), p, np.abs(gy))
    assert (np.abs(gx - wx) <= 1e-5 * ax + 1e-7).all()
    assert (np.abs(gk - wk) <= 1e-5 * ak + 1e-7).all()


@pytest.mark.parametrize("b,n,cin,cout,k,p", [(3, 6, 8, 5, 4, 2), (2, 12, 64, 32, 3, 0), (64, 4, 16, 16, 3, 1),
                                               (2, 33, 72, 3, 5, 0), (3, 9, 8, 2, 7, 3)])
def test_ffma_int_exact(b, n, cin, cout, k, p):
    """Integer data: every partial sum is exact, so any summation order is bit-exact."""
    rng = np.random.default_rng(n * 7 + cin)
    x = rng.integers(-3, 4, (b, n, n, cin)).astype(np.float32)
    kk = rng.integers(-2, 3, (k, k, cin, cout)).astype(np.float32)
    g = oracle.geometry(n, k, k, p)
    gy = rng.integers(-2, 3, (b, g.out_h, g.out_w, cout)).astype(np.float32)
    wx, wk = oracle.tconv_backward(x, kk, p, gy)
    gx, gk, _ = gpu_bwd(x, kk, p, gy, math="ffma")
    np.testing.assert_array_equal(gx, wx)
    np.testing.assert_array_equal(gk, wk)


def test_f64_ffma_and_exact():
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (2, 7, 7, 5))
    kk = rng.uniform(-1, 1, (4, 3, 5, 6))
    g = oracle.geometry(7, 4, 3, 2)
    gy = rng.uniform(-1, 1, (2, g.out_h, g.out_w, 6))
    wx, wk = oracle.tconv_backward(x, kk, 2, gy)
    gx, gk, _ = gpu_bwd(x, kk, 2, gy, math="exact")
    np.testing.assert_array_equal(gx, wx)
    np.testing.assert_array_equal(gk, wk)
    gx, gk, _ = gpu_bwd(x, kk, 2, gy, math="ffma")
    assert scaled_err(gx, wx) <= 1e-13 and scaled_err(gk, wk) <= 1e-13


@pytest.mark.parametrize("b,n,cin,cout,k,p", [
    (4, 16, 512, 256, 4, 0),  # BASELINE C3 layer (reduced batch)
    (2, 8, 128, 64, 4, 2),    # DCGAN-standard 4x4, p = 2
    (3, 5, 64, 128, 3, 1),
    (2, 7, 96, 64, 5, 2),     # 25 taps, cin not a multiple of 64
    (2, 4, 256, 512, 3, 0),   # C5 layer b-like: two feature blocks of K
    (1, 3, 320, 64, 2, 1),    # gx channels over one 256 tile
    (2, 8, 128, 128, 4, 2),   # kernel grad on the pair kernel: N = 128 features
    (3, 5, 256, 256, 3, 1),
    (1, 3, 384, 128, 2, 1),   # kernel grad: second channel pair half empty
    (64, 8, 128, 128, 3, 0),  # kernel grad: pixel reduction split over units
])
def test_bf16_tensor_core_input_grad(b, n, cin, cout, k, p):
    rng = np.random.default_rng(b * 100 + n + cin)
    x = rng.integers(-3, 4, (b, n, n, cin)).astype(np.float32)
    kk = rng.integers(-2, 3, (k, k, cin, cout)).astype(np.float32)
    g = oracle.geometry(n, k, k, p)
    gy = rng.integers(-2, 3, (b, g.out_h, g.out_w, cout)).astype(np.float32)
    wx, wk = oracle.tconv_backward(x, kk, p, gy)
    gx, gk, path = gpu_bwd(x, kk, p, gy, math="bf16", dtype=torch.bfloat16)
    wpath = "tc-pair" if cin % 128 == 0 and cout % 128 == 0 else "simt-ffma"
    assert path == "bwd:tc-pair+" + wpath
    # exact fp32 sums, then one bf16 rounding of the input gradient
    np.testing.assert_array_equal(gx, oracle.bf16_round(wx.astype(np.float32)))
    np.testing.assert_array_equal(gk, wk)


@pytest.mark.parametrize("b,n,cin,cout,k,p", [(4, 16, 512, 256, 4, 0), (3, 7, 128, 64, 3, 1)])
def test_bf16_real_data(b, n, cin, cout, k, p):
    rng = np.random.default_rng(b + n + cin)
    x = oracle.bf16_round(rng.standard_normal((b, n, n, cin)).astype(np.float32))
    kk = oracle.bf16_round((rng.standard_normal((k, k, cin, cout)) * 0.02).astype(np.float32))
    g = oracle.geometry(n, k, k, p)
    gy = oracle.bf16_round(rng.standard_normal((b, g.out_h, g.out_w, cout)).astype(np.float32))
    wx, wk = oracle.tconv_backward(x, kk, p, gy)
    gx, gk, path = gpu_bwd(x, kk, p, gy, dtype=torch.bfloat16)  # auto -> bf16
    assert path.startswith("bwd:tc-pair")
    assert scaled_err(gx, wx) <= 1e-2
    assert scaled_err(gk, wk) <= 1e-4


def test_bf16_falls_back_to_simt_when_cout_is_not_a_k_block():
    rng = np.random.default_rng(9)
    x = oracle.bf16_round(rng.standard_normal((2, 6, 6, 64)).astype(np.float32))
    kk = oracle.bf16_round((rng.standard_normal((3, 3, 64, 40)) * 0.05).astype(np.float32))
    g = oracle.geometry(6, 3, 3, 0)
    gy = oracle.bf16_round(rng.standard_normal((2, g.out_h, g.out_w, 40)).astype(np.float32))
    wx, wk = oracle.tconv_backward(x, kk, 0, gy)
    gx, gk, path = gpu_bwd(x, kk, 0, gy, math="bf16", dtype=torch.bfloat16)
    assert path == "bwd:simt-ffma+simt-ffma"
    assert scaled_err(gx, wx) <= 1e-2 and scaled_err(gk, wk) <= 1e-4


def test_kernel_grad_accumulates_like_the_reference():
    """grad_kernel= accumulates (the reference's grad_ across backward calls):
    two half-batch calls == one full-batch call, bit-exact under EXACT math."""
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, (4, 5, 5, 3)).astype(np.float32)
    kk = rng.uniform(-1, 1, (3, 3, 3, 2)).astype(np.float32)
    g = oracle.geometry(5, 3, 3, 1)
    gy = rng.uniform(-1, 1, (4, g.out_h, g.out_w, 2)).astype(np.float32)
    t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    acc = torch.zeros((3, 3, 3, 2), dtype=torch.float32, device="cuda")
    for s in (slice(0, 2), slice(2, 4)):
        sc.transpose_conv_fused_backward(t(x[s]), t(kk), 1, t(gy[s]), math="exact", input_grad=False,
                                         grad_kernel=acc)
    _, wk = oracle.tconv_backward(x, kk, 1, gy)
    np.testing.assert_array_equal(acc.cpu().numpy(), wk)


def test_empty_batch_zeroes_the_kernel_grad():
    t = torch.zeros((0, 4, 4, 8), device="cuda")
    gy = torch.zeros((0, 7, 7, 4), device="cuda")
    gx, gk = sc.transpose_conv_fused_backward(t, torch.ones((3, 3, 8, 4), device="cuda"), 1, gy)
    assert tuple(gx.shape) == (0, 4, 4, 8)
    assert torch.count_nonzero(gk).item() == 0


def test_errors():
    x = torch.zeros((1, 4, 4, 2), device="cuda")
    k = torch.zeros((3, 3, 2, 2), device="cuda")
    gy = torch.zeros((1, 5, 5, 2), device="cuda")  # out = 2n + 2p - k = 5
    with pytest.raises(sc.ContractError):
        sc.transpose_conv_fused_backward(x, k, 0, torch.zeros((1, 6, 6, 2), device="cuda"))
    with pytest.raises(sc.ContractError):
        sc.transpose_conv_fused_backward(x, torch.zeros((3, 3, 3, 2), device="cuda"), 0, gy)
    with pytest.raises(sc.ContractError):
        sc.transpose_conv_fused_backward(x.bfloat16(), k.bfloat16(), 0, gy, math="exact")
    with pytest.raises(sc.ShapeError):
        sc.transpose_conv_fused_backward(torch.zeros((1, 1, 1, 2), device="cuda"),
                                         torch.zeros((7, 7, 2, 2), device="cuda"), 0,
                                         torch.zeros((1, 1, 1, 2), device="cuda"))


def test_layer_class_mirrors_the_reference_layer():
    """FusedTConv: forward caches the input, backward returns gx and accumulates
    into grad, state error before forward (reference test_netdemo.cpp:222-238)."""
    rng = np.random.default_rng(5)
    kk = rng.uniform(-1, 1, (4, 4, 3, 2))
    layer = sc.FusedTConv(torch.from_numpy(kk), 2, math="exact")
    with pytest.raises(sc.StateError):
        layer.backward(torch.zeros((1, 8, 8, 2), dtype=torch.float64, device="cuda"))
    x = rng.uniform(-1, 1, (2, 4, 4, 3))
    y = layer.forward(torch.from_numpy(x))
    np.testing.assert_array_equal(y.cpu().numpy(), oracle.tconv_fused(x, kk, 2))
    g = oracle.geometry(4, 4, 4, 2)
    gy = rng.uniform(-1, 1, (2, g.out_h, g.out_w, 2))
    gx = layer.backward(torch.from_numpy(gy).cuda())
    wx, wk = oracle.tconv_backward(x, kk, 2, gy)
    np.testing.assert_array_equal(gx.cpu().numpy(), wx)
    (vals, grads), = layer.params()
    np.testing.assert_array_equal(grads.cpu().numpy(), wk)
    layer.zero_grads()
    assert torch.count_nonzero(layer.grad).item() == 0


@pytest.mark.parametrize("n,cin,cout,k,p", [(5, 3, 4, 3, 1), (4, 2, 3, 4, 2), (6, 4, 2, 5, 3)])
def test_autograd_matches_torch_conv_transpose(n, cin, cout, k, p):
    """The autograd wrapper's gradients equal torch's conv_transpose2d gradients
    (stride 2, padding k-1-p, flipped kernel) in double."""
    rng = np.random.default_rng(n + k)
    x = torch.tensor(rng.uniform(-1, 1, (2, n, n, cin)), device="cuda", requires_grad=True)
    kk = torch.tensor(rng.uniform(-1, 1, (k, k, cin, cout)), device="cuda", requires_grad=True)
    y = sc.TransposeConvFused.apply(x, kk, p)
    gy = torch.tensor(rng.uniform(-1, 1, tuple(y.shape)), device="cuda")
    (y * gy).sum().backward()
    x2 = x.detach().clone().permute(0, 3, 1, 2).requires_grad_(True)
    w2 = kk.detach().clone().flip(0, 1).permute(2, 3, 0, 1).contiguous().requires_grad_(True)
    y2 = torch.nn.functional.conv_transpose2d(x2, w2, stride=2, padding=k - 1 - p)
    torch.testing.assert_close(y2.permute(0, 2, 3, 1), y.detach(), rtol=1e-12, atol=1e-12)
    (y2 * gy.permute(0, 3, 1, 2)).sum().backward()
    torch.testing.assert_close(x2.grad.permute(0, 2, 3, 1), x.grad, rtol=1e-12, atol=1e-12)
    torch.testing.assert_close(w2.grad.permute(2, 3, 0, 1).flip(0, 1), kk.grad, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("streamk", ["0", "1"])
@pytest.mark.parametrize("b,n,cin,cout,k,p", [(4, 16, 512, 256, 4, 0), (64, 8, 128, 128, 3, 0),
                                               (9, 5, 256, 128, 3, 1)])
def test_kernel_grad_schedules(b, n, cin, cout, k, p, streamk, monkeypatch):
    """Both kernel-gradient schedules of the pair kernel (pixel splits and the
    stream-K pieces) are bit-exact on integer data, with and without accumulate."""
    monkeypatch.setenv("SEGCONV_WGRAD_STREAMK", streamk)
    rng = np.random.default_rng(b + n + cin + int(streamk))
    x = rng.integers(-3, 4, (b, n, n, cin)).astype(np.float32)
    kk = rng.integers(-2, 3, (k, k, cin, cout)).astype(np.float32)
    g = oracle.geometry(n, k, k, p)
    gy = rng.integers(-2, 3, (b, g.out_h, g.out_w, cout)).astype(np.float32)
    _, wk = oracle.tconv_backward(x, kk, p, gy)
    t = lambda a: torch.from_numpy(a).cuda().bfloat16()  # noqa: E731
    _, gk = sc.transpose_conv_fused_backward(t(x), t(kk), p, t(gy), input_grad=False)
    assert sc.last_path() == "bwd:-+tc-pair"
    np.testing.assert_array_equal(gk.cpu().numpy(), wk)
    acc = torch.ones_like(gk)
    sc.transpose_conv_fused_backward(t(x), t(kk), p, t(gy), input_grad=False, grad_kernel=acc)
    np.testing.assert_array_equal(acc.cpu().numpy(), wk + 1)


@pytest.mark.parametrize("b,n,cin,cout,k", [(128, 16, 512, 256, 4),   # BASELINE C3, full size
                                            (1024, 5, 512, 256, 3),   # C5 layer b, full batch
                                            (1024, 7, 256, 128, 3)])  # C5 layer c, full batch
def test_full_size_tensor_core_backward_equals_simt(b, n, cin, cout, k):
    """At the BASELINE sizes (too large for the CPU oracle): on integer data every
    partial sum is exact, so the tcgen05 input/kernel gradients must equal the
    independent SIMT kernels' bit for bit (both round the same exact sums to bf16
    for the input gradient); plus linearity in the output gradient."""
    gen = torch.Generator(device="cuda").manual_seed(b + n)
    ri = lambda shape, lo, hi: torch.randint(lo, hi + 1, shape, device="cuda", generator=gen).bfloat16()  # noqa: E731
    g = sc.tconv_geometry(n, k, k, 0)
    x = ri((b, n, n, cin), -3, 3)
    kk = ri((k, k, cin, cout), -2, 2)
    gy1 = ri((b, g.out_h, g.out_w, cout), -1, 1)
    gy2 = ri((b, g.out_h, g.out_w, cout), -1, 1)
    gx_tc, gk_tc = sc.transpose_conv_fused_backward(x, kk, 0, gy1, math="bf16")
    assert sc.last_path() == "bwd:tc-pair+tc-pair"
    gx_s, gk_s = sc.transpose_conv_fused_backward(x, kk, 0, gy1, math="ffma")
    assert sc.last_path() == "bwd:simt-ffma+simt-ffma"
    assert torch.equal(gx_tc, gx_s)
    assert torch.equal(gk_tc, gk_s)
    # and against the oracle (not only CUDA vs CUDA): the input gradient of
    # sampled images depends on that image alone; exact sums rounded to bf16
    idx = [0, b - 1]
    xs, ks_, gys = (t.float().cpu().numpy() for t in (x[idx], kk, gy1[idx]))
    wx, _ = oracle.tconv_backward(xs, ks_, 0, gys)
    np.testing.assert_array_equal(gx_tc[idx].float().cpu().numpy(), oracle.bf16_round(wx))
    _, gk2 = sc.transpose_conv_fused_backward(x, kk, 0, gy2, math="bf16", input_grad=False)
    _, gk12 = sc.transpose_conv_fused_backward(x, kk, 0, (gy1.float() + gy2.float()).bfloat16(), math="bf16",
                                               input_grad=False)
    assert torch.equal(gk12, gk_tc + gk2)  # linear in the output gradient, exact


def test_bf16_narrow_output_backward():
    """bf16 layers with 3-feature outputs on wide maps take the narrow-output SIMT
    kernels (no tensor-core mode for cout < 64): bf16 input gradient within the
    bf16 bar, fp32 kernel gradient within 1e-4."""
    rng = np.random.default_rng(21)
    x = oracle.bf16_round(rng.standard_normal((1, 64, 64, 64)).astype(np.float32))
    kk = oracle.bf16_round((rng.standard_normal((5, 5, 64, 3)) * 0.05).astype(np.float32))
    g = oracle.geometry(64, 5, 5, 0)
    gy = oracle.bf16_round(rng.standard_normal((1, g.out_h, g.out_w, 3)).astype(np.float32))
    wx, wk = oracle.tconv_backward(x, kk, 0, gy)
    gx, gk, path = gpu_bwd(x, kk, 0, gy, math="bf16", dtype=torch.bfloat16)
    assert path == "bwd:simt-narrow+simt-narrow"
    assert scaled_err(gx, wx) <= 1e-2 and scaled_err(gk, wk) <= 1e-4


# ---- fp32 input gradient in split-fp16 math on the pair kernel (math="f16x3")
@pytest.mark.parametrize("b,n,cin,cout,k,p", [
    (2, 64, 64, 32, 3, 0),    # C2 shape (reduced batch): one [hi | lo] box of 64 channels per tap
    (3, 16, 128, 64, 4, 2),   # cout = 64: [hi | lo] is two boxes -> SIMT
    (2, 9, 96, 32, 5, 1),     # 5x5, p = 1: 25 taps
])
def test_f16x3_input_grad_on_tensor_cores(b, n, cin, cout, k, p):
    rng = np.random.default_rng(b * 31 + n + cin + k)
    x = rng.uniform(-1, 1, (b, n, n, cin)).astype(np.float32)
    kk = (rng.standard_normal((k, k, cin, cout)) * 0.059).astype(np.float32)
    g = oracle.geometry(n, k, k, p)
    gy = rng.uniform(-1, 1, (b, g.out_h, g.out_w, cout)).astype(np.float32)
    wx, wk = oracle.tconv_backward(x, kk, p, gy)
    gx, gk, path = gpu_bwd(x, kk, p, gy, math="f16x3")
    dpath = "tc-pair-split" if cout == 32 and k * k <= 25 else "simt-ffma"
    assert path == f"bwd:{dpath}+simt-ffma", path
    # fp32 bar (reference tensors_equal_approx) on the input gradient; the
    # kernel gradient runs FFMA
    scaled = np.abs(gx - wx) / np.maximum(np.maximum(np.abs(gx), np.abs(wx)), 1.0)
    assert scaled.max() <= 1e-5, scaled.max()
    ak = oracle.tconv_backward(np.abs(x), np.abs(kk), p, np.abs(gy))[1]
    assert (np.abs(gk - wk) <= 1e-5 * ak + 1e-7).all()


def test_f16x3_input_grad_range():
    """Large and small magnitudes: the split scales gy and the kernel by powers
    of two (max 2^14), so nothing overflows fp16 and the result keeps the bar."""
    rng = np.random.default_rng(77)
    b, n, cin, cout, k, p = 1, 16, 64, 32, 3, 0
    g = oracle.geometry(n, k, k, p)
    x = rng.uniform(-1, 1, (b, n, n, cin)).astype(np.float32)
    for gs, ws in [(1e6, 1e3), (1e-6, 1e-3), (3e4, 7e4)]:
        kk = (rng.standard_normal((k, k, cin, cout)) * ws).astype(np.float32)
        gy = (rng.uniform(-1, 1, (b, g.out_h, g.out_w, cout)) * gs).astype(np.float32)
        wx, _ = oracle.tconv_backward(x, kk, p, gy)
        gx, _, path = gpu_bwd(x, kk, p, gy, math="f16x3")
        assert path.startswith("bwd:tc-pair-split"), path
        assert np.isfinite(gx).all()
        scaled = np.abs(gx - wx) / np.maximum(np.maximum(np.abs(gx), np.abs(wx)), 1.0)
        if scaled.max() <= 1e-5:
            continue
        # ill-conditioned sums (1e9-sized products that cancel; the reference's
        # own fp32 result is then far from the exact answer): the same criterion
        # as the forward's range tests -- error against the exact (f64) answer
        # in units of each output's conditioning sum sum |g||w|, at most 4x the
        # reference's own (or 2^-20)
        exact, _ = oracle.scatter_backward_f64(x, kk, p, gy)
        cond, _ = oracle.scatter_backward_f64(np.abs(x), np.abs(kk), p, np.abs(gy))
        live = cond > 0

        def en(a):
            return float((np.abs(a - exact)[live] / cond[live]).max())
        assert en(gx) <= max(2.0 ** -20, 4 * en(wx)), (gs, ws, en(gx), en(wx))

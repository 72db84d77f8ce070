"""GPU parity of conv2d_valid (reference reference_ops.hpp:86-102)
against the C oracle pinned to the reference (tests/golden/conv_valid.npz):
the SIMT kernels for fp32 (<= 1e-5 scaled) and the tcgen05 CTA-pair kernel for
bf16 (stride-1 im2col walk over the output pixels, every tap an offset; bit-exact
on integer data up to the one bf16 output rounding)."""
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
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    assert got.shape == want.shape
    return float((np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), 1.0)).max())


def test_fp32_matches_reference_goldens():
    """Summation order differs from the reference (FMA, tiles): the bar is the fp32
    rounding bound 1e-5 * sum|x*k| per output (the goldens use unnormalised U[-1,1]
    weights, so the sums reach |y| ~ 15 with 576 terms)."""
    z = np.load(os.path.join(G, "conv_valid.npz"))
    for i in range(int(z["count"])):
        s, k = z[f"c{i}_src"], z[f"c{i}_k"]
        y = sc.conv2d_valid(torch.from_numpy(s).cuda(), torch.from_numpy(k).cuda())
        assert sc.last_path().startswith("simt")
        bound = 1e-5 * oracle.conv2d_valid(np.abs(s), np.abs(k)) + 1e-7
        assert (np.abs(y.cpu().numpy() - z[f"c{i}_y"]) <= bound).all(), i


@pytest.mark.parametrize("b,h,w,cin,kh,kw,cout", [
    (2, 9, 9, 64, 3, 3, 64),      # the conventional path of a C2-like layer (bf16)
    (3, 12, 7, 128, 4, 2, 96),    # rectangular map and kernel
    (1, 33, 33, 256, 4, 4, 128),  # C3 conventional layer on the upsampled map
    (4, 6, 5, 64, 5, 5, 72),      # 25 taps, cout not a multiple of 32
    (2, 3, 3, 512, 3, 3, 512),    # single output pixel per image, two feature tiles
])
def test_bf16_tensor_core_int_exact(b, h, w, cin, kh, kw, cout):
    rng = np.random.default_rng(b * 100 + h + cin)
    s = rng.integers(-3, 4, (b, h, w, cin)).astype(np.float32)
    k = rng.integers(-2, 3, (kh, kw, cin, cout)).astype(np.float32)
    y = sc.conv2d_valid(torch.from_numpy(s).cuda().bfloat16(), torch.from_numpy(k).cuda().bfloat16())
    assert sc.last_path() == "tc-pair"
    want = oracle.bf16_round(oracle.conv2d_valid(s, k))
    np.testing.assert_array_equal(y.float().cpu().numpy(), want)


def test_bf16_epilogue_and_real_data():
    rng = np.random.default_rng(7)
    s = oracle.bf16_round(rng.standard_normal((2, 10, 10, 128)).astype(np.float32))
    k = oracle.bf16_round((rng.standard_normal((3, 3, 128, 64)) * 0.03).astype(np.float32))
    bias = rng.uniform(-0.1, 0.1, 64).astype(np.float32)
    y = sc.conv2d_valid(torch.from_numpy(s).cuda().bfloat16(), torch.from_numpy(k).cuda().bfloat16(),
                        bias=torch.from_numpy(bias).cuda(), activation="relu")
    assert sc.last_path() == "tc-pair"
    want = np.maximum(oracle.conv2d_valid(s, k) + bias, 0)
    assert scaled_err(y.float().cpu().numpy(), want) <= 1e-2


def test_bf16_conventional_transpose_conv_uses_the_tensor_core_conv():
    """transpose_conv_naive (upsample + pad + conv2d_valid) on bf16 runs the same
    tensor-core correlation and equals the fused result on integer data."""
    rng = np.random.default_rng(11)
    x = rng.integers(-3, 4, (2, 8, 8, 128)).astype(np.float32)
    k = rng.integers(-2, 3, (4, 4, 128, 64)).astype(np.float32)
    xb, kb = torch.from_numpy(x).cuda().bfloat16(), torch.from_numpy(k).cuda().bfloat16()
    yn = sc.transpose_conv_naive(xb, kb, 2)
    assert sc.last_path() == "tc-pair"
    np.testing.assert_array_equal(yn.float().cpu().numpy(), oracle.bf16_round(oracle.tconv_fused(x, k, 2)))


# ---- backward (reference netdemo/layers.hpp:98-122, net::ConvValid::backward)
def test_backward_exact_matches_reference_goldens():
    z = np.load(os.path.join(G, "conv_valid.npz"))
    for i in range(int(z["count"])):
        t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
        gx, gk = sc.conv2d_valid_backward(t(z[f"c{i}_src"]), t(z[f"c{i}_k"]), t(z[f"c{i}_gy"]), math="exact")
        assert sc.last_path() == "bwd:simt-exact+simt-exact"
        np.testing.assert_array_equal(gx.cpu().numpy(), z[f"c{i}_gx"])
        np.testing.assert_array_equal(gk.cpu().numpy(), z[f"c{i}_gk"])


@pytest.mark.parametrize("b,h,w,cin,kh,kw,cout", [(2, 9, 7, 5, 3, 2, 4), (3, 12, 12, 64, 3, 3, 32),
                                                  (1, 6, 8, 16, 5, 5, 3), (2, 20, 20, 130, 4, 4, 70)])
def test_backward_ffma(b, h, w, cin, kh, kw, cout):
    rng = np.random.default_rng(b + h + cin)
    s = rng.uniform(-1, 1, (b, h, w, cin)).astype(np.float32)
    k = (rng.standard_normal((kh, kw, cin, cout)) * 0.05).astype(np.float32)
    gy = rng.uniform(-1, 1, (b, h - kh + 1, w - kw + 1, cout)).astype(np.float32)
    wx, wk = oracle.conv2d_valid_backward(s, k, gy)
    t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    gx, gk = sc.conv2d_valid_backward(t(s), t(k), t(gy), math="ffma")
    assert sc.last_path() == "bwd:simt-ffma+simt-ffma"
    ax, ak = oracle.conv2d_valid_backward(np.abs(s), np.abs(k), np.abs(gy))
    assert (np.abs(gx.cpu().numpy() - wx) <= 1e-5 * ax + 1e-7).all()
    assert (np.abs(gk.cpu().numpy() - wk) <= 1e-5 * ak + 1e-7).all()


@pytest.mark.parametrize("b,h,w,cin,kh,kw,cout", [(2, 9, 9, 128, 3, 3, 128), (3, 12, 7, 256, 4, 2, 128),
                                                  (1, 33, 33, 256, 4, 4, 256), (4, 6, 5, 128, 5, 5, 64)])
def test_backward_bf16_tensor_core_int_exact(b, h, w, cin, kh, kw, cout):
    rng = np.random.default_rng(b * 10 + h + cin)
    s = rng.integers(-3, 4, (b, h, w, cin)).astype(np.float32)
    k = rng.integers(-2, 3, (kh, kw, cin, cout)).astype(np.float32)
    gy = rng.integers(-2, 3, (b, h - kh + 1, w - kw + 1, cout)).astype(np.float32)
    wx, wk = oracle.conv2d_valid_backward(s, k, gy)
    t = lambda a: torch.from_numpy(a).cuda().bfloat16()  # noqa: E731
    gx, gk = sc.conv2d_valid_backward(t(s), t(k), t(gy))
    wpath = "tc-pair" if cin % 128 == 0 and cout % 128 == 0 else "simt-ffma"
    assert sc.last_path() == "bwd:tc-pair+" + wpath
    np.testing.assert_array_equal(gx.float().cpu().numpy(), oracle.bf16_round(wx))
    np.testing.assert_array_equal(gk.cpu().numpy(), wk)


def test_conventional_training_path_matches_the_fused_backward():
    """The reference's conventional model (Upsample2x -> pad -> ConvValid) trained on
    the GPU: upsample2x_pad_backward(conv2d_valid_backward(...)) gives the same input
    and kernel gradients as the fused layer's backward (exact, integer data)."""
    rng = np.random.default_rng(21)
    for (n, cin, cout, k, p) in [(6, 8, 5, 4, 2), (5, 3, 2, 3, 1), (7, 4, 4, 5, 0)]:
        x = rng.integers(-3, 4, (2, n, n, cin)).astype(np.float32)
        kk = rng.integers(-2, 3, (k, k, cin, cout)).astype(np.float32)
        g = oracle.geometry(n, k, k, p)
        gy = rng.integers(-2, 3, (2, g.out_h, g.out_w, cout)).astype(np.float32)
        t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
        up = sc.upsample2x_pad(t(x), p)
        gup, gk = sc.conv2d_valid_backward(up, t(kk), t(gy), math="exact")
        gx = sc.upsample2x_pad_backward(gup, n, p)
        assert sc.last_path() == "simt-gather"
        wx, wk = oracle.tconv_backward(x, kk, p, gy)
        np.testing.assert_array_equal(gx.cpu().numpy(), wx)
        np.testing.assert_array_equal(gk.cpu().numpy(), wk)


def test_conventional_model_layers_train_like_the_fused_layer():
    """Python mirrors of the reference netdemo layers: Upsample2x -> ConvValid
    (the conventional model) and FusedTConv give identical outputs and gradients
    on integer data (reference test_netdemo.cpp compares the two models)."""
    rng = np.random.default_rng(33)
    n, cin, cout, k, p = 6, 4, 3, 4, 2
    x = torch.from_numpy(rng.integers(-3, 4, (2, n, n, cin)).astype(np.float64))
    kk = torch.from_numpy(rng.integers(-2, 3, (k, k, cin, cout)).astype(np.float64))
    up, conv = sc.Upsample2x(p), sc.ConvValid(kk, math="exact")
    fused = sc.FusedTConv(kk, p, math="exact")
    y1 = conv.forward(up.forward(x))
    y2 = fused.forward(x)
    assert torch.equal(y1, y2)
    g = torch.from_numpy(rng.integers(-2, 3, tuple(y1.shape)).astype(np.float64)).cuda()
    gx1 = up.backward(conv.backward(g))
    gx2 = fused.backward(g)
    assert torch.equal(gx1, gx2)
    assert torch.equal(conv.grad, fused.grad)
    with pytest.raises(sc.StateError):
        sc.ConvValid(kk).backward(g)

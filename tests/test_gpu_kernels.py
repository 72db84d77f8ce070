"""Per-kernel-family GPU parity: each tcgen05 kernel the dispatcher picks is
exercised at small sizes (ragged batches, partial tiles, tile/segment edges,
fused epilogues) against the C oracle, and the test asserts which kernel ran
(segconv_last_path).

Bars: split-fp16 math on fp32 data -> the reference's
tensors_equal_approx at 1e-5; bf16 operand paths -> 1e-2 (the oracle sees the
same bf16-rounded inputs, so the remaining difference is fp32 summation order,
<= 1e-4 here, plus bf16 output rounding where the output is bf16).
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2209_03704_b200 import segconv as sc

pytestmark = pytest.mark.gpu
TOL_F32 = 1e-5
TOL_TC = 1e-2


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")


def scaled_err(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape
    return float((np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), 1.0)).max())


def run(x, k, p, math, act=None, bias=None, out_dtype=None):
    dt = torch.bfloat16 if math == "bf16" else torch.float32
    g = sc.tconv_geometry(x.shape[1], k.shape[0], k.shape[1], p)
    sks = sc.segregate(torch.from_numpy(k).cuda().to(dt), p, math=math)
    bt = torch.from_numpy(bias).cuda() if bias is not None else None
    y = sc.transpose_conv_fused(torch.from_numpy(x).cuda().to(dt), sks, g, activation=act, bias=bt,
                                out_dtype=out_dtype)
    torch.cuda.synchronize()
    return y.float().cpu().numpy(), sc.last_path()


def want_of(x, k, p, act=None, bias=None):
    w = oracle.tconv_fused(x, k, p)
    if bias is not None:
        w = w + bias
    if act == "relu":
        w = np.maximum(w, 0)
    if act == "tanh":
        w = np.tanh(w)
    return w


# ---- fp32 64 -> 32, 3x3 (BASELINE C2 family): TMEM-weight fold kernel
@pytest.mark.parametrize("batch,n,act", [(1, 64, None), (3, 64, "relu"), (2, 40, "tanh"), (5, 17, None)])
def test_fold_ts_split_fp16(batch, n, act):
    rng = np.random.default_rng(batch * 100 + n)
    x = rng.uniform(-1, 1, (batch, n, n, 64)).astype(np.float32)
    k = (rng.standard_normal((3, 3, 64, 32)) * 0.059).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, 32).astype(np.float32) if act else None
    got, path = run(x, k, 0, "f16x3", act, b)
    assert path == "tc-fold-ts"
    assert scaled_err(got, want_of(x, k, 0, act, b)) <= TOL_F32


# other shapes the anchors-on-M fold kernel takes: cout < 32 (per-element
# stores), cin = 32 (one stage per unit), p = 1 and k = 4 (other class / shift
# sets: the column order search), bf16 output, bias + activation
@pytest.mark.parametrize("batch,n,cin,cout,k,p,act,odt", [
    (2, 33, 64, 20, 3, 0, "relu", None),
    (3, 30, 32, 32, 3, 0, None, None),
    (2, 31, 64, 32, 3, 1, "tanh", None),
    (2, 24, 64, 24, 4, 1, None, None),
    (2, 40, 64, 32, 3, 0, "relu", torch.bfloat16),
])
def test_fold_ts_shapes(batch, n, cin, cout, k, p, act, odt):
    rng = np.random.default_rng(batch * 1000 + n * 10 + cout + k)
    x = rng.uniform(-1, 1, (batch, n, n, cin)).astype(np.float32)
    w = (rng.standard_normal((k, k, cin, cout)) * 0.06).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, cout).astype(np.float32) if act else None
    got, path = run(x, w, p, "f16x3", act, b, out_dtype=odt)
    assert path == "tc-fold-ts", path
    want = want_of(x, w, p, act, b)
    assert scaled_err(got, want) <= (1e-2 if odt is not None else TOL_F32)


# ---- wide bf16 layers (C3, C5 a-c): CTA-pair kernel
@pytest.mark.parametrize("batch,n,cin,cout,ks,act", [
    (4, 16, 512, 256, 4, None),   # C3 shape (reduced batch)
    (3, 4, 1024, 512, 3, "relu"),  # C5 layer a: two feature tiles, tiny images
    (2, 7, 256, 128, 3, "relu"),   # C5 layer c
    (5, 5, 512, 256, 3, None),     # odd image, partial pair tile
    (2, 9, 64, 96, 4, "tanh"),     # cout not a multiple of 64, single k-block
    (2, 6, 192, 128, 3, "relu"),   # cin % 128 != 0: one k-block per pipeline stage
    (3, 6, 128, 128, 3, None),     # two k-blocks per stage, a single stage per tap
])
def test_pair_kernel_bf16(batch, n, cin, cout, ks, act):
    rng = np.random.default_rng(batch * 7 + n + cin)
    x = oracle.bf16_round(rng.standard_normal((batch, n, n, cin)).astype(np.float32))
    k = oracle.bf16_round((rng.standard_normal((ks, ks, cin, cout)) * 0.02).astype(np.float32))
    got, path = run(x, k, 0, "bf16", act, out_dtype=torch.float32)
    assert path == "tc-pair"
    assert scaled_err(got, want_of(x, k, 0, act)) <= 1e-4  # fp32 accumulate; bar is 1e-2


@pytest.mark.parametrize("batch,n,cin,cout,ks,p,act", [
    (2, 16, 128, 64, 4, 2, "relu"),  # DCGAN-standard layer: 4x4, out = 2N (p = 2, p_fused = 1)
    (3, 5, 256, 128, 3, 1, None),    # p = 1: odd-padding class swap, p_fused = 0
    (2, 8, 64, 64, 4, 3, None),      # p = 3: p_fused = 1, odd parity
    (1, 7, 128, 96, 5, 2, "tanh"),   # 5x5, p = 2
    (4, 4, 512, 256, 4, 2, "relu"),  # GAN first layer 4 -> 8
])
def test_pair_kernel_padded(batch, n, cin, cout, ks, p, act):
    """p_orig > 0: the padded grid is staged by 4-D TMA boxes whose
    out-of-image part is zero-filled."""
    rng = np.random.default_rng(batch * 31 + n + cin + p)
    x = oracle.bf16_round(rng.standard_normal((batch, n, n, cin)).astype(np.float32))
    k = oracle.bf16_round((rng.standard_normal((ks, ks, cin, cout)) * 0.02).astype(np.float32))
    got, path = run(x, k, p, "bf16", act, out_dtype=torch.float32)
    assert path == "tc-pair"
    assert scaled_err(got, want_of(x, k, p, act)) <= 1e-4


@pytest.mark.parametrize("batch,n,cin,cout,ks,p", [(4, 16, 512, 256, 4, 0), (2, 16, 128, 64, 4, 2),
                                                    (3, 5, 256, 128, 3, 1)])
def test_pair_kernel_halo_shift_staging(batch, n, cin, cout, ks, p, monkeypatch):
    """The halo-shift staging of the pair kernel (linear TMA rows for p_fused = 0,
    padded 4-D boxes otherwise) -- the alternative to im2col, selected by
    SEGCONV_WIDE_IM2COL=0."""
    monkeypatch.setenv("SEGCONV_WIDE_IM2COL", "0")
    rng = np.random.default_rng(batch * 3 + n + p)
    x = oracle.bf16_round(rng.standard_normal((batch, n, n, cin)).astype(np.float32))
    k = oracle.bf16_round((rng.standard_normal((ks, ks, cin, cout)) * 0.02).astype(np.float32))
    got, path = run(x, k, p, "bf16", out_dtype=torch.float32)
    assert path == "tc-pair"
    assert scaled_err(got, want_of(x, k, p)) <= 1e-4


def test_pair_kernel_bf16_output():
    rng = np.random.default_rng(5)
    x = oracle.bf16_round(rng.standard_normal((2, 16, 16, 128)).astype(np.float32))
    k = oracle.bf16_round((rng.standard_normal((4, 4, 128, 64)) * 0.02).astype(np.float32))
    got, path = run(x, k, 0, "bf16")
    assert path == "tc-pair"
    assert scaled_err(got, want_of(x, k, 0)) <= TOL_TC


# ---- high-resolution 5x5 -> 3 fp32 (C4 family): pixel-scatter row-ring kernel
@pytest.mark.parametrize("batch,n,cin,act,bias", [(1, 128, 64, None, False), (2, 128, 64, "tanh", True),
                                                  (3, 256, 32, None, False), (1, 256, 64, "tanh", False)])
def test_ring_kernel(batch, n, cin, act, bias):
    rng = np.random.default_rng(batch * 13 + n + cin)
    x = rng.uniform(-1, 1, (batch, n, n, cin)).astype(np.float32)
    k = (rng.standard_normal((5, 5, cin, 3)) * 0.02).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, 3).astype(np.float32) if bias else None
    got, path = run(x, k, 0, "f16x3", act, b)
    assert path == "tc-ring"
    assert scaled_err(got, want_of(x, k, 0, act, b)) <= TOL_F32


def test_ring_falls_back_for_other_sizes():
    """The row ring needs 128- or 256-pixel rows; other sizes take the folded kernel."""
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (2, 40, 40, 64)).astype(np.float32)
    k = (rng.standard_normal((5, 5, 64, 3)) * 0.02).astype(np.float32)
    got, path = run(x, k, 0, "f16x3")
    assert path == "tc-fold"
    assert scaled_err(got, want_of(x, k, 0)) <= TOL_F32


# ---- small-image 3x3 -> 3 bf16 (C5 layer d family): pixel-scatter tile kernel
@pytest.mark.parametrize("batch,n,cin,act,odt", [(4, 11, 128, "tanh", torch.float32),
                                                 (3, 7, 64, None, torch.float32),
                                                 (7, 11, 128, "tanh", torch.bfloat16),
                                                 (2, 30, 192, None, torch.float32),
                                                 (1, 3, 64, "relu", torch.float32)])
def test_tile_kernel(batch, n, cin, act, odt):
    rng = np.random.default_rng(batch * 17 + n + cin)
    x = oracle.bf16_round(rng.standard_normal((batch, n, n, cin)).astype(np.float32))
    k = oracle.bf16_round((rng.standard_normal((3, 3, cin, 3)) * 0.02).astype(np.float32))
    got, path = run(x, k, 0, "bf16", act, out_dtype=odt)
    assert path == "tc-tile"
    tol = 1e-4 if odt == torch.float32 else TOL_TC
    assert scaled_err(got, want_of(x, k, 0, act)) <= tol


# ---- integer-valued data: every kernel family is bit-exact
def _ints(rng, shape, lo, hi):
    return rng.integers(lo, hi + 1, shape).astype(np.float32)


@pytest.mark.parametrize("case", [
    # (math, batch, n, cin, cout, k, p, expected path)
    ("f16x3", 3, 64, 64, 32, 3, 0, "tc-fold-ts"),
    ("f16x3", 2, 128, 64, 3, 5, 0, "tc-ring"),
    ("bf16", 5, 11, 128, 3, 3, 0, "tc-tile"),
    ("bf16", 4, 8, 128, 128, 4, 0, "tc-pair"),
    ("bf16", 3, 6, 64, 64, 4, 2, "tc-pair"),
    ("bf16", 2, 5, 256, 96, 3, 1, "tc-pair"),
])
def test_kernel_families_int_exact(case):
    math, batch, n, cin, cout, ks, p, path = case
    rng = np.random.default_rng(batch * 1000 + n * 10 + ks)
    x = _ints(rng, (batch, n, n, cin), -3, 3)
    k = _ints(rng, (ks, ks, cin, cout), -2, 2)
    got, ran = run(x, k, p, math, out_dtype=torch.float32)
    assert ran == path
    want = oracle.tconv_fused(x, k, p)
    assert np.array_equal(got, want), f"max abs diff {np.abs(got - want).max()}"


@pytest.mark.parametrize("math,shape", [("f16x3", (64, 64, 32, 3)), ("bf16", (11, 128, 3, 3)),
                                        ("bf16", (16, 512, 256, 4))])
def test_empty_batch_is_a_no_op(math, shape):
    """batch == 0 (the reference's empty-tensor edge): no launch, empty result."""
    n, cin, cout, ks = shape
    dt = torch.bfloat16 if math == "bf16" else torch.float32
    g = sc.tconv_geometry(n, ks, ks, 0)
    sks = sc.segregate(torch.zeros((ks, ks, cin, cout), device="cuda", dtype=dt), 0, math=math)
    y = sc.transpose_conv_fused(torch.zeros((0, n, n, cin), device="cuda", dtype=dt), sks, g)
    assert tuple(y.shape) == (0, g.out_h, g.out_w, cout)


@pytest.mark.parametrize("n,p", [(128, 2), (130, 0)])
def test_pair_kernel_large_maps(n, p):
    """Maps wider than the halo-shift staging's TMA box (EB-GAN's last layer,
    128 x 128 x 64 -> 256 x 256 x 64, 4x4, p = 2): the im2col path has no such
    limit, so AUTO must not refuse them."""
    rng = np.random.default_rng(n + p)
    x = rng.integers(-2, 3, (1, n, n, 64)).astype(np.float32)
    k = rng.integers(-1, 2, (4, 4, 64, 64)).astype(np.float32)
    got, path = run(x, k, p, "bf16", out_dtype=torch.float32)
    assert path == "tc-pair"
    assert np.array_equal(got, oracle.tconv_fused(x, k, p))


@pytest.mark.parametrize("batch,n,cin,cout,p,act,path", [
    (4, 32, 128, 3, 2, "tanh", "tc-tile"),   # DCGAN / Art-GAN last layer (4x4, out = 2N)
    (3, 32, 64, 3, 2, "tanh", "tc-tile"),    # GP-GAN last layer
    (2, 50, 64, 3, 2, None, "tc-pair"),      # too wide for a 128-pixel scatter tile
    (2, 9, 128, 40, 1, None, "tc-pair"),     # 33..63 features: one 64-wide tile
    (2, 6, 64, 17, 3, "relu", "tc-pair"),
])
def test_narrow_outputs_at_padding(batch, n, cin, cout, p, act, path):
    """cout < 64 with p_fused > 0: the 3-channel 4x4 layers take the pixel-scatter
    tile kernel (input offsets shifted by -p/2, out-of-image taps masked), others
    the pair kernel with a 32- or 64-wide feature tile; integer data, exact."""
    rng = np.random.default_rng(batch + n + cout)
    x = rng.integers(-2, 3, (batch, n, n, cin)).astype(np.float32)
    k = rng.integers(-1, 2, (4, 4, cin, cout)).astype(np.float32)
    got, ran = run(x, k, p, "bf16", act, out_dtype=torch.float32)
    assert ran == path
    want = want_of(x, k, p, act)
    if act == "tanh":
        assert np.abs(got - want).max() <= 1e-6
    else:
        assert np.array_equal(got, want)


@pytest.mark.parametrize("batch,n,cin,p,odt", [(5, 8, 64, 0, torch.float32), (3, 16, 128, 2, torch.bfloat16),
                                               (2, 21, 192, 2, torch.float32), (7, 5, 64, 2, torch.float32),
                                               (3, 8, 256, 2, torch.bfloat16), (2, 9, 512, 2, torch.float32)])
def test_tile_kernel_4x4(batch, n, cin, p, odt):
    """4x4 -> 3 on the tile kernel: p = 0 (folded panels) and even p > 0 (K-major
    panels with the tile image appended); bf16 real data, tolerance as C5 d.
    cin 256 / 512: the weight image leaves room for one CTA per SM only."""
    rng = np.random.default_rng(batch * 3 + n + p)
    x = oracle.bf16_round(rng.standard_normal((batch, n, n, cin)).astype(np.float32))
    k = oracle.bf16_round((rng.standard_normal((4, 4, cin, 3)) * 0.02).astype(np.float32))
    got, path = run(x, k, p, "bf16", "tanh", out_dtype=odt)
    assert path == "tc-tile"
    tol = 1e-4 if odt == torch.float32 else TOL_TC
    assert scaled_err(got, want_of(x, k, p, "tanh")) <= tol


def test_tile_kernel_not_used_where_class_grids_exceed_the_input():
    """4x4 at p = 4: out = 2n + 4, class grids of n + 2 rows -- not n x n anchors."""
    rng = np.random.default_rng(44)
    x = rng.integers(-2, 3, (2, 10, 10, 64)).astype(np.float32)
    k = rng.integers(-1, 2, (4, 4, 64, 3)).astype(np.float32)
    got, path = run(x, k, 4, "bf16", out_dtype=torch.float32)
    assert path != "tc-tile"
    assert np.array_equal(got, oracle.tconv_fused(x, k, 4))


@pytest.mark.parametrize("batch,n,cin,cout,ks,p,act", [
    (4, 16, 512, 256, 4, 0, None),    # BASELINE C3 shape in fp32: main product 4 x 512 / 16 = 128 steps
    (2, 8, 128, 64, 4, 2, "relu"),    # DCGAN layer in fp32
    (3, 5, 256, 128, 3, 1, "tanh"),
    (2, 7, 64, 96, 3, 0, None),
    (2, 4, 768, 256, 3, 0, None),     # 4 taps x 768 / 16 = 192 steps, the AUTO limit
])
def test_pair_kernel_fp32_split(batch, n, cin, cout, ks, p, act):
    """fp32 wide layers (the reference's own dtype) on the pair kernel: x and w as
    fp16 [hi | lo] halves, three MMA passes (xh.wh, xl.wh, xh.wl).  Bar: 1e-5
    scaled against the reference order, or -- where the reference's own fp32
    sums (2048 terms for C3) already miss the exact f64 answer by that much --
    at least as close to the exact answer as the reference is (within 2x), as
    test_gpu_parity does for FFMA."""
    rng = np.random.default_rng(batch + n + cin + p)
    x = rng.uniform(-1, 1, (batch, n, n, cin)).astype(np.float32)
    k = (rng.standard_normal((ks, ks, cin, cout)) / np.sqrt(cin * ks * ks)).astype(np.float32)
    got, path = run(x, k, p, "f16x3", act)
    assert path == "tc-pair"
    want = want_of(x, k, p, act)
    if scaled_err(got, want) > TOL_F32:
        exact = oracle.tconv_fused(x.astype(np.float64), k.astype(np.float64), p)
        if act == "relu":
            exact = np.maximum(exact, 0)
        if act == "tanh":
            exact = np.tanh(exact)
        assert scaled_err(got, exact) <= max(TOL_F32, 2 * scaled_err(want, exact))


def test_pair_kernel_fp32_split_int_exact():
    rng = np.random.default_rng(77)
    x = rng.integers(-3, 4, (2, 8, 8, 128)).astype(np.float32)
    k = rng.integers(-2, 3, (4, 4, 128, 64)).astype(np.float32)
    got, path = run(x, k, 2, "f16x3")
    assert path == "tc-pair"
    assert np.array_equal(got, oracle.tconv_fused(x, k, 2))


def test_fp32_long_k_layers_stay_on_ffma_under_auto():
    """AUTO keeps fp32 layers whose main tensor-core accumulation would take > 192
    K-steps (4 taps x 1024 channels / 16 = 256) on FFMA, which meets 1e-5; the
    explicit f16x3 request still runs the pair kernel, within ~4e-8 per step."""
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (2, 4, 4, 1024)).astype(np.float32)
    k = (rng.standard_normal((4, 4, 1024, 128)) / np.sqrt(1024 * 16)).astype(np.float32)
    g = sc.tconv_geometry(4, 4, 4, 0)
    xt, kt = torch.from_numpy(x).cuda(), torch.from_numpy(k).cuda()
    y = sc.transpose_conv_fused(xt, sc.segregate(kt, 0), g).cpu().numpy()
    assert sc.last_path().startswith("simt")
    want = oracle.tconv_fused(x, k, 0)
    assert scaled_err(y, want) <= TOL_F32
    y2 = sc.transpose_conv_fused(xt, sc.segregate(kt, 0, math="f16x3"), g).cpu().numpy()
    assert sc.last_path() == "tc-pair"
    assert scaled_err(y2, want) <= 256 * 4e-8 + TOL_F32


@pytest.mark.parametrize("cin,cout,ks", [(512, 32, 3), (256, 16, 5)])
def test_fp32_narrow_long_k_layers_leave_the_folded_kernel(cin, cout, ks):
    """The folded kernels keep every product in one accumulator over the union
    window; when that would take > 192 accumulation steps AUTO moves the layer to
    the pair kernel's split mode (main product apart), which meets 1e-5."""
    rng = np.random.default_rng(cin + ks)
    x = rng.uniform(-1, 1, (2, 12, 12, cin)).astype(np.float32)
    k = (rng.standard_normal((ks, ks, cin, cout)) / np.sqrt(cin * ks * ks)).astype(np.float32)
    g = sc.tconv_geometry(12, ks, ks, 0)
    y = sc.transpose_conv_fused(torch.from_numpy(x).cuda(), torch.from_numpy(k).cuda(), 0).cpu().numpy()
    assert sc.last_path() == "tc-pair"
    assert scaled_err(y, oracle.tconv_fused(x, k, 0)) <= TOL_F32


@pytest.mark.parametrize("batch,n,cin,cout,ks,p,act", [
    (4, 16, 512, 256, 4, 0, None),    # C3 shape in fp32, tf32 tensor cores
    (2, 8, 128, 64, 4, 2, "relu"),
    (3, 5, 256, 96, 3, 1, "tanh"),
])
def test_pair_kernel_tf32(batch, n, cin, cout, ks, p, act):
    """math="tf32" (explicit; AUTO keeps fp32 at the 1e-5 bar): fp32 operands on
    kind::tf32 MMAs, 32 channels per 128-byte row; bar 1e-2 as the bf16 paths."""
    rng = np.random.default_rng(batch * 9 + n + cin)
    x = rng.uniform(-1, 1, (batch, n, n, cin)).astype(np.float32)
    k = (rng.standard_normal((ks, ks, cin, cout)) / np.sqrt(cin * ks * ks)).astype(np.float32)
    got, path = run(x, k, p, "tf32", act)
    assert path == "tc-pair"
    assert scaled_err(got, want_of(x, k, p, act)) <= TOL_TC
    xi = rng.integers(-3, 4, (batch, n, n, cin)).astype(np.float32)
    ki = rng.integers(-2, 3, (ks, ks, cin, cout)).astype(np.float32)
    got, _ = run(xi, ki, p, "tf32")
    assert np.array_equal(got, oracle.tconv_fused(xi, ki, p))  # small integers are exact in tf32


@pytest.mark.parametrize("math,batch,cin,cout,ks,p", [
    ("bf16", 24, 64, 128, 4, 0),    # 4 classes x 19 pair tiles = 76 units on 74 pairs: 2 split
    ("bf16", 24, 64, 256, 4, 0),    # NT = 256 halves
    ("bf16", 12, 64, 384, 4, 0),    # two feature tiles, the second one split
    ("f16x3", 24, 64, 128, 4, 0),   # split-fp16 passes on half tiles
    ("tf32", 24, 64, 128, 4, 0),
])
def test_pair_kernel_tail_half_tiles(math, batch, cin, cout, ks, p):
    """The pair kernel runs the units of a last, partial wave as feature half-tiles
    (N = NT / 2, two pairs per unit) when they fit twice over: every output
    feature of those units must still be written once, exactly."""
    rng = np.random.default_rng(batch + cout)
    x = rng.integers(-3, 4, (batch, 16, 16, cin)).astype(np.float32)
    k = rng.integers(-2, 3, (ks, ks, cin, cout)).astype(np.float32)
    got, path = run(x, k, p, math, out_dtype=torch.float32)
    assert path == "tc-pair"
    assert np.array_equal(got, oracle.tconv_fused(x, k, p))


@pytest.mark.parametrize("batch,n,cin,cout,p", [
    (2, 64, 64, 64, 2),     # EB-GAN 64 -> 128 layer shape: 2-D column blocks, four class accumulators
    (1, 128, 64, 64, 2),    # 128-wide map: blocks narrower than the padded row
    (2, 72, 128, 48, 2),    # two k-blocks, a partial feature tile
    (1, 66, 64, 64, 3),     # p = 3: odd parity classes
])
def test_pair_kernel_all_class_halo(batch, n, cin, cout, p):
    """Narrow outputs on large padded maps take the halo staging with all four
    classes per unit (ALLQ) and 2-D column blocks: bit-exact on integer data."""
    rng = np.random.default_rng(n * 3 + cin + p)
    x = rng.integers(-3, 4, (batch, n, n, cin)).astype(np.float32)
    k = rng.integers(-2, 3, (4, 4, cin, cout)).astype(np.float32)
    got, path = run(x, k, p, "bf16", out_dtype=torch.float32)
    assert path == "tc-pair"
    assert np.array_equal(got, oracle.tconv_fused(x, k, p))
    xr = oracle.bf16_round(rng.standard_normal((batch, n, n, cin)).astype(np.float32))
    kr = oracle.bf16_round((rng.standard_normal((4, 4, cin, cout)) * 0.05).astype(np.float32))
    got, _ = run(xr, kr, p, "bf16", "relu", out_dtype=torch.float32)
    assert scaled_err(got, want_of(xr, kr, p, "relu")) <= 1e-4


@pytest.mark.parametrize("n,cin,cout,p", [(16, 128, 64, 2), (64, 64, 64, 2), (8, 256, 128, 0)])
def test_pair_kernel_bf16_output_tanh(n, cin, cout, p):
    """bf16 outputs take the hardware tanh (error ~2^-11, below bf16 rounding)."""
    rng = np.random.default_rng(n + cin + cout)
    x = oracle.bf16_round(rng.standard_normal((2, n, n, cin)).astype(np.float32))
    k = oracle.bf16_round((rng.standard_normal((4, 4, cin, cout)) * 0.05).astype(np.float32))
    got, path = run(x, k, p, "bf16", "tanh")
    assert path == "tc-pair"
    assert scaled_err(got, want_of(x, k, p, "tanh")) <= TOL_TC


# ---- tiny layers (BASELINE C1 family): one thread per output, unrolled class taps
@pytest.mark.parametrize("batch,n,cin,cout,k,p,dt", [
    (1, 32, 1, 1, 3, 0, torch.float32),   # C1
    (3, 17, 1, 2, 7, 2, torch.float32),   # 4 x 4 taps per class, padding
    (2, 12, 2, 3, 5, 1, torch.float32),   # cin > 1: the channel-loop form
    (2, 20, 1, 1, 4, 1, torch.bfloat16),  # bf16 storage
])
def test_tiny_layer_kernel(batch, n, cin, cout, k, p, dt):
    rng = np.random.default_rng(n * 10 + k + cin)
    x = rng.uniform(-1, 1, (batch, n, n, cin)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, cin, cout)).astype(np.float32)
    if dt == torch.bfloat16:
        x, w = oracle.bf16_round(x), oracle.bf16_round(w)
    g = sc.tconv_geometry(n, k, k, p)
    sks = sc.segregate(torch.from_numpy(w).cuda().to(dt), p, math="ffma")
    y = sc.transpose_conv_fused(torch.from_numpy(x).cuda().to(dt), sks, g, math="ffma")
    torch.cuda.synchronize()
    assert sc.last_path() == "simt-tiled", sc.last_path()
    want = oracle.tconv_fused(x, w, p)
    tol = 1e-2 if dt == torch.bfloat16 else 1e-5
    assert scaled_err(y.float().cpu().numpy(), want) <= tol

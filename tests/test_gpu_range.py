"""Range guard of the split-fp16 (f16x3) tensor-core path, the default (AUTO)
math for fp32 layers.  The reference accepts every finite float
(tensor.hpp:79-96); fp16 halves do not (max 65504, subnormal floor 2^-24).
Weights are power-of-two scaled at segregate time, activations are range-
checked by the converter warps and a CTA that saw an out-of-range value
recomputes its outputs with FFMA (paper_2209_03704_b200/csrc/tc_guard.cuh);
the pair kernel's fp32 mode scales x by a power of two instead.  Every case:
AUTO, finite output, within the fp32 bar of the oracle, on the kernel family
the shape normally takes (the guard must not change dispatch)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2209_03704_b200 import segconv as sc

pytestmark = pytest.mark.gpu


def scaled_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float((np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)).max())


def rel_err(a, b):
    """error relative to the largest output (meaningful when |y| << 1)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def assert_fp32_bar(got, x, k, p):
    """The fp32 bar: within 1e-5 (scaled, and relative to the largest output)
    of the reference's fp32 result.  Where that fails because the problem is
    ill-conditioned (1e11-sized products whose sums cancel: the reference's own
    fp32 result is then percents away from the exact answer), the result must
    be as accurate as fp32 summation is: its error against the exact (f64
    scatter) answer, in units of the conditioning sum A = sum |x||w| of each
    output, at most 4x the reference's own (or 2^-20)."""
    ref = oracle.tconv_fused(x, k, p)
    if scaled_err(got, ref) <= 1e-5 and rel_err(got, ref) <= 1e-5:
        return
    exact = oracle.scatter_f64(x.astype(np.float64), k.astype(np.float64), p)
    cond = oracle.scatter_f64(np.abs(x).astype(np.float64), np.abs(k).astype(np.float64), p)
    live = cond > 0
    assert np.all(got[~live] == 0)

    def en(a):
        return float((np.abs(a.astype(np.float64) - exact)[live] / cond[live]).max())
    assert en(got) <= max(2.0 ** -20, 4 * en(ref)), (en(got), en(ref))


def run_auto(x, k, p, act=None):
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    kt = torch.from_numpy(np.ascontiguousarray(k)).cuda()
    y = sc.transpose_conv_fused(xt, kt, p, activation=act)
    torch.cuda.synchronize()
    return y.cpu().numpy(), sc.last_path()


# (name, batch, n, cin, cout, k, p, expected AUTO path)
SHAPES = [
    ("C2", 2, 64, 64, 32, 3, 0, "tc-fold-ts"),
    ("C4", 1, 256, 64, 3, 5, 0, "tc-ring"),
    ("fold", 2, 20, 64, 8, 3, 0, "tc-fold"),
    ("fold-block", 1, 80, 32, 4, 4, 1, "tc-fold"),
    ("pair-split", 2, 8, 128, 64, 4, 0, "tc-pair"),
]
# (x scale, w scale): overflow of x, overflow of w, tiny x under huge w
# (the small check), tiny w (exponent scaling), ordinary data
RANGES = [(1e6, 1e5), (1.0, 1e7), (1e-6, 1e5), (1.0, 1e-30), (1.0, 0.05)]


@pytest.mark.parametrize("xs,ws", RANGES)
@pytest.mark.parametrize("shape", SHAPES, ids=[s[0] for s in SHAPES])
def test_auto_f16x3_any_finite_range(shape, xs, ws):
    name, b, n, cin, cout, kk, p, path = shape
    rng = np.random.default_rng(hash((name, xs, ws)) % 2**32)
    x = (rng.uniform(-1, 1, (b, n, n, cin)) * xs).astype(np.float32)
    k = (rng.standard_normal((kk, kk, cin, cout)) * ws).astype(np.float32)
    got, used = run_auto(x, k, p)
    assert used == path, used
    assert np.isfinite(got).all()
    assert_fp32_bar(got, x, k, p)


def test_guard_fallback_only_in_the_bad_cta():
    """One out-of-range element in an otherwise ordinary C2-shaped batch: the
    outputs far from it still come from the tensor-core path (bit pattern of a
    clean run), the ones it touches are right."""
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, (2, 64, 64, 64)).astype(np.float32)
    k = (rng.standard_normal((3, 3, 64, 32)) * 0.06).astype(np.float32)
    clean, _ = run_auto(x, k, 0)
    x2 = x.copy()
    x2[1, 40, 17, 5] = 3.0e6
    got, used = run_auto(x2, k, 0)
    assert used == "tc-fold-ts"
    assert np.isfinite(got).all()
    assert_fp32_bar(got, x2, k, 0)
    np.testing.assert_array_equal(got[0], clean[0])  # image 0 is in other CTAs entirely


def test_tanh_epilogue_with_scaled_weights():
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, (1, 256, 256, 64)).astype(np.float32)
    k = (rng.standard_normal((5, 5, 64, 3)) * 3e-9).astype(np.float32)
    got, used = run_auto(x, k, 0, act="tanh")
    assert used == "tc-ring"
    want = np.tanh(oracle.tconv_fused(x, k, 0))
    assert rel_err(got, want) <= 1e-5

"""Pins the CPU oracle (oracle/segconv_oracle.c) against golden vectors made by
the reference itself (tests/golden/make_golden.py).  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _npz(name):
    return np.load(os.path.join(G, name))


def test_geometry_table_matches_reference():
    # reference proj/tests/test_geometry.cpp:9-70
    for row in json.load(open(os.path.join(G, "geometry.json"))):
        args = row["args"]
        if row["ok"]:
            g = oracle.geometry(*args)
            assert list(g.__dict__.values()) == [bool(v) if i >= 9 else v
                                                 for i, v in enumerate(row["g"])], args
        else:
            with pytest.raises(oracle.OracleError) as e:
                oracle.geometry(*args)
            assert e.value.code == 1  # ShapeError


def test_geometry_closed_form():
    for n in range(1, 13):
        for k in range(1, 8):
            for p in range(0, 5):
                out = 2 * n + 2 * p - k
                if out < 1:
                    continue
                g = oracle.geometry(n, k, k, p)
                assert g.out_h == g.out_w == out
                assert g.up_h == 2 * n - 1 + 2 * p and g.p_fused == p // 2
                assert g.trim_extra_row == (k % 2 == 1) == g.trim_extra_col
    g = oracle.geometry(8, 3, 4, 2)
    assert (g.out_h, g.out_w, g.trim_extra_row, g.trim_extra_col) == (17, 16, True, False)


def test_tap_arithmetic():
    # reference proj/tests/test_segregation.cpp:24-51
    assert [oracle.first_active_tap(p, r) for p, r in [(0, 0), (0, 1), (1, 0), (1, 1), (2, 0), (3, 1)]] \
        == [0, 1, 1, 0, 0, 0]
    for n in range(1, 10):
        for p in range(6):
            assert oracle.active_tap_count(n, p, 0) + oracle.active_tap_count(n, p, 1) == n
    assert oracle.active_tap_count(5, 0, 0) == 3 and oracle.active_tap_count(5, 0, 1) == 2
    assert oracle.active_tap_count(1, 0, 1) == 0
    for p in range(7):
        for r in range(2):
            assert oracle.class_input_offset(p, r) == (r if p % 2 == 0 else 0)


def test_segregation_matches_reference():
    z = _npz("segregation.npz")
    keys = sorted({k.rsplit("_", 1)[0] for k in z.files if k.endswith("_kernel")})
    assert keys
    for key in keys:
        k = z[key + "_kernel"]
        p = int(key.split("_p")[1])
        subs = oracle.segregate(k, p)
        _, offs = oracle.subkernel_dims(k.shape[0], k.shape[1], p)
        for q in range(4):
            np.testing.assert_array_equal(subs[q], z[f"{key}_sub{q}"])
        assert [tuple(o) for o in z[key + "_offs"]] == offs


def test_segregation_routing_goldens():
    # iota 3x3 p=2: (0,0)={1,3,7,9}, (0,1)={2,8}, (1,0)={4,6}, (1,1)={5}
    k = np.arange(1, 10, dtype=np.float32).reshape(3, 3, 1, 1)
    s = oracle.segregate(k, 2)
    assert s[0].ravel().tolist() == [1, 3, 7, 9]
    assert s[1].ravel().tolist() == [2, 8]
    assert s[2].ravel().tolist() == [4, 6]
    assert s[3].ravel().tolist() == [5]
    # odd padding swaps classes diagonally (test_segregation.cpp:90-107)
    so = oracle.segregate(k, 1)
    for q in range(4):
        np.testing.assert_array_equal(so[q], s[3 - q])


def test_frozen_worked_example():
    z = _npz("frozen.npz")
    want = np.array([[1, 1, 3, 2, 2], [1, 1, 3, 2, 2], [4, 4, 10, 6, 6], [3, 3, 7, 4, 4],
                     [3, 3, 7, 4, 4]], dtype=np.float32)
    np.testing.assert_array_equal(z["naive"][..., 0], want)
    np.testing.assert_array_equal(oracle.tconv_fused(z["x"], z["k"], 2), z["fused"])
    np.testing.assert_array_equal(oracle.tconv_naive(z["x"], z["k"], 2), z["naive"])


def test_verify_cases_bit_exact():
    """All 200 run_verify cases (seed 20240911): oracle fused == reference naive, exactly."""
    z = _npz("verify_cases.npz")
    summ = z["summary"]
    assert summ[0] == 200 and summ[1] == 0          # reference fuzz clean
    assert summ[4] == 1 and summ[5] == 4            # injected fault localised to case 4
    for i in range(200):
        n, k, p, cin, cout = z[f"c{i}_dims"].tolist()
        x = z[f"c{i}_x"].astype(np.float32)
        kern = z[f"c{i}_k"].astype(np.float32)
        want = z[f"c{i}_y"]
        got = oracle.tconv_fused(x, kern, p)
        assert got.shape == want.shape
        np.testing.assert_array_equal(got, want, err_msg=f"case {i}")
        np.testing.assert_array_equal(oracle.tconv_naive(x, kern, p), want)


def test_real_cases_bit_exact():
    """U[-1,1] cases: the oracle reproduces the reference's fused AND naive outputs bit for bit."""
    z = _npz("real_cases.npz")
    for i in range(int(z["count"])):
        b, n, cin, cout, kh, kw, p = z[f"r{i}_dims"].tolist()
        x, k = z[f"r{i}_x"], z[f"r{i}_k"]
        np.testing.assert_array_equal(oracle.tconv_fused(x, k, p), z[f"r{i}_fused"])
        np.testing.assert_array_equal(oracle.tconv_naive(x, k, p), z[f"r{i}_naive"])


def test_double_precision_case():
    z = _npz("f64_case.npz")
    np.testing.assert_array_equal(oracle.tconv_fused(z["x"], z["k"], 2), z["fused"])
    np.testing.assert_array_equal(oracle.tconv_naive(z["x"], z["k"], 2), z["naive"])


def test_scatter_agrees_on_int_cases():
    # reference proj/tests/test_reference_ops.cpp:114-134
    z = _npz("verify_cases.npz")
    for i in range(0, 200, 5):
        n, k, p, cin, cout = z[f"c{i}_dims"].tolist()
        got = oracle.scatter_f64(z[f"c{i}_x"].astype(np.float64), z[f"c{i}_k"].astype(np.float64), p)
        np.testing.assert_array_equal(got, z[f"c{i}_y"].astype(np.float64))


def test_counts_match_reference():
    for row in json.load(open(os.path.join(G, "counts.json"))):
        assert list(oracle.count_ops(*row["shape"])) == row["ops"], row["shape"]


def test_baseline_useful_macs():
    # SURVEY.md 8(a) a13
    per = {(32, 1, 1, 3, 3, 0): 8464, (64, 64, 32, 3, 3, 0): 1158152192 // 16,
           (16, 512, 256, 4, 4, 0): 52613349376 // 128, (256, 64, 3, 5, 5, 0): 9878470656 // 32}
    for s, v in per.items():
        assert oracle.count_ops(*s)[2] == v


@pytest.mark.skipif(not oracle.ref_available(), reason="reference shim not built")
def test_reference_shim_live():
    """Where the reference shim exists, the oracle agrees with it live on fresh inputs."""
    rng = np.random.default_rng(7)
    for (n, cin, cout, k, p) in [(5, 3, 4, 3, 0), (6, 2, 5, 4, 1), (3, 1, 1, 5, 3), (7, 4, 17, 2, 2)]:
        x = rng.uniform(-1, 1, (2, n, n, cin)).astype(np.float32)
        kk = rng.uniform(-1, 1, (k, k, cin, cout)).astype(np.float32)
        np.testing.assert_array_equal(oracle.tconv_fused(x, kk, p), oracle.ref_tconv_fused(x, kk, p))
        np.testing.assert_array_equal(oracle.ref_tconv_fused_parallel(x, kk, p, 3),
                                      oracle.ref_tconv_fused(x, kk, p))


# ---------------------------------------------------------------- backward
def _bwd_cases():
    z = _npz("backward.npz")
    for i in range(int(z["count"])):
        yield i, [int(v) for v in z[f"b{i}_dims"]], z[f"b{i}_x"], z[f"b{i}_k"], z[f"b{i}_gy"], \
            z[f"b{i}_gx"], z[f"b{i}_gk"]


def test_backward_bit_exact_vs_reference_goldens():
    """oracle.tconv_backward == net::FusedTConv::backward (layers.hpp:171-211), bit for bit,
    float and double, batches with the kernel gradient summed over images."""
    n_cases = 0
    for i, dims, x, k, gy, gx, gk in _bwd_cases():
        p = dims[6]
        got_x, got_k = oracle.tconv_backward(x, k, p, gy)
        assert got_x.dtype == gx.dtype
        np.testing.assert_array_equal(got_x, gx, err_msg=f"case {i} dims {dims}")
        np.testing.assert_array_equal(got_k, gk, err_msg=f"case {i} dims {dims}")
        n_cases += 1
    assert n_cases >= 25


def test_backward_matches_independent_scatter_form():
    """The scatter-form gradients (sharing no code with the restatement) agree in double."""
    for i, dims, x, k, gy, gx, gk in _bwd_cases():
        sx, sk = oracle.scatter_backward_f64(x, k, dims[6], gy)
        tol = 1e-12 if x.dtype == np.float64 else 1e-4
        np.testing.assert_allclose(sx, gx, rtol=0, atol=tol * max(1.0, np.abs(sx).max()))
        np.testing.assert_allclose(sk, gk, rtol=0, atol=tol * max(1.0, np.abs(sk).max()))


@pytest.mark.parametrize("n,cin,cout,k,p", [(3, 1, 2, 3, 0), (4, 2, 1, 4, 2), (3, 2, 3, 5, 3),
                                             (4, 1, 1, 1, 1)])
def test_backward_finite_differences(n, cin, cout, k, p):
    """Central differences of L = sum(G * fused(x, k)) confirm both gradients
    (the reference's own check, tests/test_netdemo.cpp:55-101,137-152)."""
    rng = np.random.default_rng(n * 100 + k * 10 + p)
    x = rng.uniform(-1, 1, (1, n, n, cin))
    kk = rng.uniform(-1, 1, (k, k, cin, cout))
    g = oracle.geometry(n, k, k, p)
    G = rng.uniform(-1, 1, (1, g.out_h, g.out_w, cout))
    gx, gk = oracle.tconv_backward(x, kk, p, G)
    eps = 1e-6

    def loss(xx, kk2):
        return float((oracle.tconv_fused(xx, kk2, p) * G).sum())

    for arr, grad, is_x in ((x, gx, True), (kk, gk, False)):
        flat = arr.reshape(-1)
        for e in range(flat.size):
            s = flat[e]
            flat[e] = s + eps
            lp = loss(x, kk)
            flat[e] = s - eps
            lm = loss(x, kk)
            flat[e] = s
            fd = (lp - lm) / (2 * eps)
            assert abs(fd - grad.reshape(-1)[e]) <= 1e-6 * max(1.0, abs(fd)), (is_x, e)


@pytest.mark.skipif(not oracle.ref_available(), reason="reference shim not built")
def test_backward_reference_live():
    rng = np.random.default_rng(11)
    for (b, n, cin, cout, k, p) in [(2, 5, 3, 4, 3, 0), (3, 6, 2, 5, 4, 2), (1, 3, 1, 1, 5, 3)]:
        x = rng.uniform(-1, 1, (b, n, n, cin)).astype(np.float32)
        kk = rng.uniform(-1, 1, (k, k, cin, cout)).astype(np.float32)
        g = oracle.geometry(n, k, k, p)
        gy = rng.uniform(-1, 1, (b, g.out_h, g.out_w, cout)).astype(np.float32)
        a = oracle.tconv_backward(x, kk, p, gy)
        r = oracle.ref_tconv_backward(x, kk, p, gy)
        np.testing.assert_array_equal(a[0], r[0])
        np.testing.assert_array_equal(a[1], r[1])
        gx, gk, secs = oracle.ref_time_backward(x, kk, p, gy, 2)
        np.testing.assert_array_equal(gx, r[0])
        np.testing.assert_allclose(gk, r[1], rtol=0, atol=1e-5)
        assert secs >= 0


def test_conv2d_valid_bit_exact_vs_reference_goldens():
    """oracle.conv2d_valid == reference conv2d_valid (reference_ops.hpp:86-102)."""
    z = _npz("conv_valid.npz")
    for i in range(int(z["count"])):
        np.testing.assert_array_equal(oracle.conv2d_valid(z[f"c{i}_src"], z[f"c{i}_k"]), z[f"c{i}_y"])


def test_conv2d_valid_backward_bit_exact_vs_reference_goldens():
    """oracle.conv2d_valid_backward == net::ConvValid::backward (layers.hpp:98-122)."""
    z = _npz("conv_valid.npz")
    for i in range(int(z["count"])):
        gx, gk = oracle.conv2d_valid_backward(z[f"c{i}_src"], z[f"c{i}_k"], z[f"c{i}_gy"])
        np.testing.assert_array_equal(gx, z[f"c{i}_gx"])
        np.testing.assert_array_equal(gk, z[f"c{i}_gk"])

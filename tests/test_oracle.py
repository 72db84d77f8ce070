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

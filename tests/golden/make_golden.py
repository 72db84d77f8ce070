"""Generates tests/golden/* from the REFERENCE itself (oracle/_ref shim over the
unmodified /root/reference headers).  Run in the build container:

    make -C oracle && python tests/golden/make_golden.py

Fixtures (all small):
  geometry.json      tconv_geometry over n<=12, k<=7, p<=4 + rect cases
                     (reference proj/tests/test_geometry.cpp:9-70)
  counts.json        count_ops_naive/fused for BASELINE configs and tests
                     (proj/include/segconv/analysis.hpp:31-67)
  segregation.npz    sub-kernels of iota kernels (proj/tests/test_segregation.cpp)
  frozen.npz         2x2 input, 3x3 ones, p=2 worked example
                     (proj/tests/test_reference_ops.cpp:96-112)
  verify_cases.npz   the first 200 run_verify cases, seed 20240911 (inputs +
                     reference outputs; proj/include/segconv/verify.hpp:66-125)
  real_cases.npz     U[-1,1] float cases incl. BASELINE-shaped reductions, with
                     the reference's fused and naive outputs
  f64_case.npz       a double-precision case (proj/tests/test_fused.cpp:61-70)
  backward.npz       input and kernel gradients of net::FusedTConv (forward +
                     backward per image, grads zeroed once per batch;
                     proj/include/segconv/netdemo/layers.hpp:171-211) on the
                     FD-test shape family (proj/tests/test_netdemo.cpp:137-152),
                     rectangular kernels, batches, integer and double cases
                     (`python tests/golden/make_golden.py backward` rewrites
                     only this file)
  conv_valid.npz     conv2d_valid (reference_ops.hpp:86-102) on rectangular
                     maps and kernels, and net::ConvValid's gradients
                     (netdemo/layers.hpp:98-122) (`python tests/golden/make_golden.py conv`)
  sgc/*.sgc          SGC1 tensor files written by the reference's save_tensor
                     (tensor_io.hpp:93-103) + sgc/values.npz with their contents
                     (`python tests/golden/make_golden.py sgc`)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def iota(kh, kw, cin=1, cout=1):
    return np.arange(1, kh * kw * cin * cout + 1, dtype=np.float32).reshape(kh, kw, cin, cout)


def main():
    # ---------------------------------------------------------------- geometry
    geo = []
    for n in range(1, 13):
        for k in range(1, 8):
            for p in range(0, 5):
                try:
                    g = oracle.ref_geometry(n, k, k, p)
                    geo.append({"args": [n, k, k, p], "ok": True, "g": list(g.__dict__.values())})
                except oracle.OracleError as e:
                    geo.append({"args": [n, k, k, p], "ok": False, "code": e.code})
    for args in ([8, 3, 4, 2], [28, 5, 5, 0], [0, 3, 3, 1], [4, 0, 3, 1], [4, 3, 3, -1],
                 [1, 3, 3, 0], [32, 3, 3, 0], [64, 3, 3, 0], [16, 4, 4, 0], [256, 5, 5, 0],
                 [4, 3, 3, 0], [5, 3, 3, 0], [7, 3, 3, 0], [11, 3, 3, 0]):
        try:
            g = oracle.ref_geometry(*args)
            geo.append({"args": args, "ok": True, "g": list(g.__dict__.values())})
        except oracle.OracleError as e:
            geo.append({"args": args, "ok": False, "code": e.code})
    with open(os.path.join(OUT, "geometry.json"), "w") as f:
        json.dump(geo, f)

    # ------------------------------------------------------------------ counts
    shapes = [  # (n, cin, cout, kh, kw, p)
        (32, 1, 1, 3, 3, 0), (64, 64, 32, 3, 3, 0), (16, 512, 256, 4, 4, 0),
        (256, 64, 3, 5, 5, 0), (4, 1024, 512, 3, 3, 0), (5, 512, 256, 3, 3, 0),
        (7, 256, 128, 3, 3, 0), (11, 128, 3, 3, 3, 0), (224, 3, 1, 5, 5, 3),
        (4, 1024, 512, 4, 4, 2), (8, 512, 256, 4, 4, 2), (16, 256, 128, 4, 4, 2),
        (32, 128, 3, 4, 4, 2), (6, 2, 3, 4, 4, 2), (5, 3, 2, 3, 3, 1), (7, 1, 2, 5, 5, 2),
        (4, 2, 2, 7, 7, 3), (3, 2, 1, 1, 1, 0), (5, 2, 2, 3, 4, 2),
    ]
    counts = [{"shape": s, "ops": list(oracle.ref_count_ops(*s))} for s in shapes]
    with open(os.path.join(OUT, "counts.json"), "w") as f:
        json.dump(counts, f)

    # ------------------------------------------------------------- segregation
    seg = {}
    for (kh, kw, cin, cout, p) in [(3, 3, 1, 1, 2), (3, 3, 1, 1, 1), (4, 4, 1, 1, 2),
                                   (1, 1, 2, 3, 0), (5, 5, 2, 2, 3), (3, 4, 2, 3, 0),
                                   (7, 2, 1, 2, 5), (5, 5, 1, 1, 0)]:
        k = iota(kh, kw, cin, cout)
        subs, offs = oracle.ref_segregate(k, p)
        key = f"k{kh}x{kw}x{cin}x{cout}_p{p}"
        seg[key + "_kernel"] = k
        for q, s in enumerate(subs):
            seg[f"{key}_sub{q}"] = s
        seg[key + "_offs"] = np.array(offs, dtype=np.int32)
    np.savez_compressed(os.path.join(OUT, "segregation.npz"), **seg)

    # ------------------------------------------------------------------ frozen
    x = np.array([1, 2, 3, 4], dtype=np.float32).reshape(2, 2, 1)
    k = np.ones((3, 3, 1, 1), dtype=np.float32)
    np.savez_compressed(os.path.join(OUT, "frozen.npz"), x=x, k=k, p=np.int32(2),
                        naive=oracle.ref_tconv_naive(x, k, 2), fused=oracle.ref_tconv_fused(x, k, 2))

    # ------------------------------------------------------------ verify cases
    seed = 20240911
    vc = {}
    for i in range(200):
        c = oracle.ref_verify_case(seed, i)
        vc[f"c{i}_dims"] = np.array([c["n"], c["k"], c["p"], c["cin"], c["cout"]], dtype=np.int32)
        vc[f"c{i}_x"] = c["x"].astype(np.int8)
        vc[f"c{i}_k"] = c["kernel"].astype(np.int8)
        vc[f"c{i}_y"] = c["y"]
    summary = oracle.ref_run_verify(200, seed, -1)
    fault = oracle.ref_run_verify(10, seed, 4)
    vc["summary"] = np.array([summary["cases_run"], summary["failures"], summary["first_failure"],
                              fault["cases_run"], fault["failures"], fault["first_failure"]],
                             dtype=np.int32)
    np.savez_compressed(os.path.join(OUT, "verify_cases.npz"), **vc)

    # -------------------------------------------------------------- real cases
    rng = np.random.default_rng(424242)
    rc = {}
    specs = []
    for _ in range(60):
        n = int(rng.integers(1, 9))
        p = int(rng.integers(0, 5))
        cap = min(7, 2 * n - 1 + 2 * p)
        kh, kw = int(rng.integers(1, cap + 1)), int(rng.integers(1, cap + 1))
        if 2 * n + 2 * p - kh < 1 or 2 * n + 2 * p - kw < 1:
            continue
        specs.append((1, n, int(rng.integers(1, 5)), int(rng.integers(1, 5)), kh, kw, p))
    # BASELINE-shaped cases (full C1; the others reduced in batch / extent)
    specs += [(1, 32, 1, 1, 3, 3, 0), (2, 12, 64, 32, 3, 3, 0), (1, 6, 128, 64, 4, 4, 0),
              (1, 20, 64, 3, 5, 5, 0), (2, 4, 64, 32, 3, 3, 0), (2, 5, 32, 16, 3, 3, 0),
              (1, 7, 16, 8, 3, 3, 0), (1, 11, 128, 3, 3, 3, 0), (1, 9, 2, 37, 3, 3, 1)]
    for i, (b, n, cin, cout, kh, kw, p) in enumerate(specs):
        x = rng.uniform(-1, 1, (b, n, n, cin)).astype(np.float32)
        k = rng.uniform(-1, 1, (kh, kw, cin, cout)).astype(np.float32)
        rc[f"r{i}_dims"] = np.array([b, n, cin, cout, kh, kw, p], dtype=np.int32)
        rc[f"r{i}_x"] = x
        rc[f"r{i}_k"] = k
        rc[f"r{i}_fused"] = oracle.ref_tconv_fused(x, k, p)
        rc[f"r{i}_naive"] = oracle.ref_tconv_naive(x, k, p)
    rc["count"] = np.int32(len(specs))
    np.savez_compressed(os.path.join(OUT, "real_cases.npz"), **rc)

    # ---------------------------------------------------------------- double
    r64 = np.random.default_rng(9)
    x = r64.uniform(-1, 1, (6, 6, 2))
    k = r64.uniform(-1, 1, (5, 5, 2, 3))
    np.savez_compressed(os.path.join(OUT, "f64_case.npz"), x=x, k=k, p=np.int32(2),
                        fused=oracle.ref_tconv_fused(x, k, 2), naive=oracle.ref_tconv_naive(x, k, 2))
    backward()
    sgc()
    conv()
    print("golden fixtures written to", OUT)


def backward():
    rng = np.random.default_rng(137152)
    specs = []  # (batch, n, cin, cout, kh, kw, p, kind)
    while len(specs) < 20:  # the FD-test family: n 3-6, p 0-3, k 1-5, cin 1-2, cout 1-3
        n, p, k = int(rng.integers(3, 7)), int(rng.integers(0, 4)), int(rng.integers(1, 6))
        if 2 * n + 2 * p - k < 1 or k > 2 * n - 1 + 2 * p:
            continue
        specs.append((1, n, int(rng.integers(1, 3)), int(rng.integers(1, 4)), k, k, p, "real"))
    specs += [(3, 5, 3, 2, 3, 4, 2, "real"), (2, 4, 2, 3, 4, 3, 1, "real"), (4, 6, 4, 5, 4, 4, 2, "real"),
              (2, 8, 16, 8, 3, 3, 0, "real"), (3, 4, 32, 16, 4, 4, 0, "real"), (2, 5, 8, 8, 5, 5, 3, "real"),
              (3, 6, 8, 4, 4, 4, 2, "int"), (2, 5, 6, 3, 3, 3, 1, "int"), (2, 5, 2, 3, 5, 5, 2, "f64")]
    out = {"count": np.int32(len(specs))}
    for i, (b, n, cin, cout, kh, kw, p, kind) in enumerate(specs):
        g = oracle.ref_geometry(n, kh, kw, p)
        if kind == "int":
            x = rng.integers(-3, 4, (b, n, n, cin)).astype(np.float32)
            k = rng.integers(-2, 3, (kh, kw, cin, cout)).astype(np.float32)
            gy = rng.integers(-2, 3, (b, g.out_h, g.out_w, cout)).astype(np.float32)
        else:
            dt = np.float64 if kind == "f64" else np.float32
            x = rng.uniform(-1, 1, (b, n, n, cin)).astype(dt)
            k = rng.uniform(-1, 1, (kh, kw, cin, cout)).astype(dt)
            gy = rng.uniform(-1, 1, (b, g.out_h, g.out_w, cout)).astype(dt)
        gx, gk = oracle.ref_tconv_backward(x, k, p, gy)
        out[f"b{i}_dims"] = np.array([b, n, cin, cout, kh, kw, p], dtype=np.int32)
        out[f"b{i}_x"], out[f"b{i}_k"], out[f"b{i}_gy"] = x, k, gy
        out[f"b{i}_gx"], out[f"b{i}_gk"] = gx, gk
    np.savez_compressed(os.path.join(OUT, "backward.npz"), **out)


def conv():
    rng = np.random.default_rng(86102)
    out = {}
    specs = [(1, 5, 5, 1, 3, 3, 1), (2, 7, 9, 3, 3, 2, 4), (3, 6, 4, 8, 2, 3, 5), (1, 9, 9, 16, 5, 5, 7),
             (2, 4, 6, 2, 4, 1, 3), (1, 12, 10, 64, 3, 3, 32)]
    for i, (b, h, w, cin, kh, kw, cout) in enumerate(specs):
        s = rng.uniform(-1, 1, (b, h, w, cin)).astype(np.float32)
        k = rng.uniform(-1, 1, (kh, kw, cin, cout)).astype(np.float32)
        out[f"c{i}_src"], out[f"c{i}_k"] = s, k
        out[f"c{i}_y"] = oracle.ref_conv2d_valid(s, k)
        gy = rng.uniform(-1, 1, out[f"c{i}_y"].shape).astype(np.float32)
        out[f"c{i}_gy"] = gy
        out[f"c{i}_gx"], out[f"c{i}_gk"] = oracle.ref_conv2d_valid_backward(s, k, gy)
    out["count"] = np.int32(len(specs))
    np.savez_compressed(os.path.join(OUT, "conv_valid.npz"), **out)


def sgc():
    d = os.path.join(OUT, "sgc")
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng(4490)
    vals = {
        "f32_5x4x3": rng.uniform(-2, 2, (5, 4, 3)).astype(np.float32),
        "f64_2x3x2": rng.uniform(-2, 2, (2, 3, 2)),
        "f32_1x1x1": np.array([[[3.5]]], dtype=np.float32),
        "f32_6x6x8": rng.standard_normal((6, 6, 8)).astype(np.float32),
    }
    for name, v in vals.items():
        oracle.ref_save_tensor(os.path.join(d, name + ".sgc"), v)
    np.savez_compressed(os.path.join(d, "values.npz"), **vals)


if __name__ == "__main__":
    if sys.argv[1:] == ["backward"]:
        backward()
    elif sys.argv[1:] == ["sgc"]:
        sgc()
    elif sys.argv[1:] == ["conv"]:
        conv()
    else:
        main()

"""CPU-only tests of the C ABI boundary: the library loads, exports every symbol
include/segconv_b200.h declares, and its host-side logic (geometry, parity
math, sub-kernel descriptors, op counts, contract checks that fire before any
launch) matches the reference goldens.  No kernel is launched here."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

import oracle
from paper_2209_03704_b200 import _capi as A
from paper_2209_03704_b200 import segconv as sc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "tests", "golden")


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "segconv_b200.h")).read()
    declared = set(re.findall(r"\b(segconv_[a-z0-9_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    lib = A.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared but not exported"
    assert declared <= set(A.SIGNATURES), declared - set(A.SIGNATURES)


def test_geometry_matches_reference_goldens():
    for row in json.load(open(os.path.join(G, "geometry.json"))):
        args = row["args"]
        if row["ok"]:
            g = sc.tconv_geometry(*args)
            want = [bool(v) if i >= 9 else v for i, v in enumerate(row["g"])]
            assert list(g.__dict__.values()) == want, args
        else:
            with pytest.raises(sc.ShapeError):
                sc.tconv_geometry(*args)


def test_parity_helpers_match_oracle():
    for n in range(1, 10):
        for p in range(0, 7):
            for r in range(2):
                assert sc.first_active_tap(p, r) == oracle.first_active_tap(p, r)
                assert sc.active_tap_count(n, p, r) == oracle.active_tap_count(n, p, r)
                assert sc.class_input_offset(p, r) == oracle.class_input_offset(p, r)


def test_sub_kernel_dims_recipe():
    assert sc.sub_kernel_dims(5) == [(3, 3), (3, 2), (2, 3), (2, 2)]
    assert sc.sub_kernel_dims(3)[0] == (2, 2) and sc.sub_kernel_dims(3)[3] == (1, 1)
    assert sc.sub_kernel_dims(1)[3] == (0, 0)
    for bad in (4, 0):
        with pytest.raises(sc.ContractError):
            sc.sub_kernel_dims(bad)


def test_subkernel_descriptor_matches_oracle():
    for (kh, kw, cin, cout, p) in [(3, 3, 1, 1, 2), (4, 4, 512, 256, 0), (5, 5, 64, 3, 0),
                                   (1, 1, 2, 3, 0), (7, 2, 3, 5, 5), (3, 4, 2, 2, 1)]:
        for layout in (A.PANEL_REF, A.PANEL_KMAJOR):
            d = A.SubKernels()
            assert A.lib().segconv_subkernels_init(kh, kw, cin, cout, p, A.F32, layout,
                                                   C.byref(d)) == A.OK
            dims, offs = oracle.subkernel_dims(kh, kw, p)
            cpad = cout if layout == A.PANEL_REF else (cout + 15) // 16 * 16
            off = 0
            for q in range(4):
                assert (d.sub_kh[q], d.sub_kw[q]) == dims[q]
                assert (d.off_r[q], d.off_c[q]) == offs[q]
                assert d.sub_offset[q] == off
                off += dims[q][0] * dims[q][1] * cin * cpad
            assert d.total_elems == off and d.cout_pad == cpad
            assert d.p_orig_parity == p % 2


def test_subkernel_init_errors_mirror_segregate():
    d = A.SubKernels()
    assert A.lib().segconv_subkernels_init(0, 3, 1, 1, 0, A.F32, 0, C.byref(d)) == A.E_CONTRACT
    assert A.lib().segconv_subkernels_init(3, 3, 1, 1, -1, A.F32, 0, C.byref(d)) == A.E_CONTRACT
    assert A.lib().segconv_subkernels_init(3, 3, 0, 1, 0, A.F32, 0, C.byref(d)) == A.E_SHAPE


def test_counts_match_reference():
    for row in json.load(open(os.path.join(G, "counts.json"))):
        n, cin, cout, kh, kw, p = row["shape"]
        s = sc.LayerShape(n, cin, cout, kh, kw, p)
        a, b = sc.count_ops_naive(s), sc.count_ops_fused(s)
        assert [a.mults, a.adds, b.mults, b.adds] == row["ops"], row["shape"]


def _desc(kh, kw, cin, cout, p, layout=A.PANEL_REF):
    d = A.SubKernels()
    assert A.lib().segconv_subkernels_init(kh, kw, cin, cout, p, A.F32, layout, C.byref(d)) == 0
    return d


def _geom(n, kh, kw, p):
    g = A.Geometry()
    assert A.lib().segconv_tconv_geometry(n, kh, kw, p, C.byref(g)) == 0
    return g


def _fused(d, g, n, cin, batch=0, epi=0, bias=None, math=A.MATH_FFMA):
    return A.lib().segconv_transpose_conv_fused(None, A.F32, batch, n, cin, C.byref(d), None,
                                                C.byref(g), bias, epi, math, None, A.F32, None)


def test_fused_contract_checks_fire_before_launch():
    """check_fused_args (reference fused_tconv.hpp:17-35), all host-side."""
    d, g = _desc(4, 4, 2, 2, 2), _geom(6, 4, 4, 2)
    assert _fused(d, g, 6, 2) == A.OK  # batch 0: nothing to launch
    # padding parity mismatch
    assert _fused(_desc(4, 4, 2, 2, 1), g, 6, 2) == A.E_CONTRACT
    assert "parity" in A.last_error()
    # geometry built for another size
    assert _fused(d, _geom(5, 4, 4, 2), 6, 2) == A.E_CONTRACT
    # channel mismatch
    assert _fused(d, g, 6, 3) == A.E_CONTRACT
    assert "channel" in A.last_error()
    # kernel dims differ from geometry
    assert _fused(_desc(3, 3, 2, 2, 2), g, 6, 2) == A.E_CONTRACT
    # bias flag without pointer; relu+tanh together
    assert _fused(d, g, 6, 2, epi=A.EPI_BIAS) == A.E_CONTRACT
    assert _fused(d, g, 6, 2, epi=A.EPI_RELU | A.EPI_TANH) == A.E_CONTRACT
    # tensor-core math with reference-layout panels
    assert _fused(d, g, 6, 2, batch=1, math=A.MATH_BF16) == A.E_CONTRACT


def test_naive_and_conv_contract_checks():
    L = A.lib()
    # workspace too small
    assert L.segconv_transpose_conv_naive(None, A.F32, 1, 4, 2, None, 3, 3, 1, 1, None, 0, None,
                                          0, 0, None, None) == A.E_CONTRACT
    # kernel exceeds upsampled extent
    assert L.segconv_transpose_conv_naive(None, A.F32, 1, 4, 2, None, 9, 9, 1, 0, None, 0, None,
                                          0, 0, None, None) == A.E_SHAPE
    assert L.segconv_conv2d_valid(None, A.F32, 1, 3, 3, 2, None, 4, 1, 1, None, 0, 0, None,
                                  None) == A.E_SHAPE
    assert L.segconv_naive_workspace_bytes(A.F32, 32, 256, 64, 0) == 32 * 511 * 511 * 64 * 4


def test_python_mirror_validation_without_gpu():
    import torch
    k = torch.zeros(3, 3, 1, 1)
    with pytest.raises(sc.ContractError):
        sc.segregate(k, -1)
    with pytest.raises(sc.ContractError):
        sc.segregate(torch.zeros(0, 3, 1, 1), 0)
    with pytest.raises(sc.ContractError):
        sc.transpose_conv_fused_parallel(torch.zeros(4, 4, 1), None, None, 0)


def test_tensor_comparators():
    import torch
    a = torch.tensor([0.0, 1.0, -2.0])
    b = torch.tensor([-0.0, 1.0, -2.0])
    assert sc.tensors_equal_exact(a, b)          # +0 == -0
    assert not sc.tensors_equal_exact(a, b[:2])
    assert sc.tensors_equal_approx(torch.tensor([100.0]), torch.tensor([100.0005]), 1e-5)
    assert not sc.tensors_equal_approx(torch.tensor([0.5]), torch.tensor([0.50002]), 1e-5)

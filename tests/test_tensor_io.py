"""SGC1 tensor container (reference tensor_io.hpp:12-103) through the C ABI:
files written by the reference itself (tests/golden/sgc) load exactly, our
writer is byte-identical to the reference's, and malformed files fail with the
reference's error kinds and byte offsets (reference tests/test_io.cpp:44-127).
Host-only: runs without a GPU except the marked upload test."""
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2209_03704_b200 import segconv as sc

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sgc")
VALS = np.load(os.path.join(G, "values.npz"))


def test_reference_written_files_load_exactly():
    for name in VALS.files:
        want = VALS[name]
        path = os.path.join(G, name + ".sgc")
        info = sc.peek_tensor_file(path)
        assert (info.height, info.width, info.channels) == want.shape
        assert info.precision == ("f64" if want.dtype == np.float64 else "f32")
        got = sc.load_tensor(path)
        np.testing.assert_array_equal(got.numpy(), want)


def test_writer_is_byte_identical_to_the_reference(tmp_path):
    for name in VALS.files:
        path = tmp_path / (name + ".sgc")
        sc.save_tensor(torch.from_numpy(VALS[name]), str(path))
        assert path.read_bytes() == open(os.path.join(G, name + ".sgc"), "rb").read()


def test_round_trip_both_precisions(tmp_path):
    rng = np.random.default_rng(1)
    for dt in (torch.float32, torch.float64):
        t = torch.from_numpy(rng.standard_normal((5, 4, 3))).to(dt)
        p = str(tmp_path / "t.sgc")
        sc.save_tensor(t, p)
        assert sc.peek_tensor_file(p) == sc.TensorFileInfo(5, 4, 3, "f32" if dt == torch.float32 else "f64")
        assert torch.equal(sc.load_tensor(p), t)


def _bytes(path, data):
    with open(path, "wb") as f:
        f.write(data)


def _hdr(*fields):
    return b"SGC1" + b"".join(int(v).to_bytes(4, "little") for v in fields)


def test_malformed_files(tmp_path):
    p = str(tmp_path / "bad.sgc")
    with pytest.raises(sc.IoError):
        sc.load_tensor(str(tmp_path / "does_not_exist.sgc"))
    sc.save_tensor(torch.zeros((1, 1, 1)), p)
    with pytest.raises(sc.ContractError):
        sc.load_tensor(p, torch.float64)
    _bytes(p, b"NOPE................")
    with pytest.raises(sc.ParseError) as e:
        sc.peek_tensor_file(p)
    assert e.value.byte_offset == 0
    _bytes(p, b"SGC1xxxx")
    with pytest.raises(sc.ParseError) as e:
        sc.peek_tensor_file(p)
    assert e.value.byte_offset == 8
    _bytes(p, _hdr(1, 1, 1, 7))
    with pytest.raises(sc.ParseError) as e:
        sc.peek_tensor_file(p)
    assert e.value.byte_offset == 16 and "precision tag 7" in str(e.value)
    sc.save_tensor(torch.zeros((2, 2, 1)), p)  # 36 bytes
    os.truncate(p, 28)
    with pytest.raises(sc.ParseError) as e:
        sc.load_tensor(p)
    assert e.value.byte_offset == 28 and "expected 36" in str(e.value)
    _bytes(p, _hdr(0, 1, 1, 0))
    with pytest.raises(sc.ParseError) as e:
        sc.peek_tensor_file(p)
    assert e.value.byte_offset == 4
    _bytes(p, _hdr(1, 1, 1, 0) + b"\0" * 8)  # payload longer than promised
    with pytest.raises(sc.ParseError) as e:
        sc.load_tensor(p)
    assert e.value.byte_offset == 24


@pytest.mark.skipif(not oracle.ref_available(), reason="reference shim not built")
def test_error_kinds_and_offsets_match_the_reference_live(tmp_path):
    p = str(tmp_path / "bad.sgc")
    cases = [b"NOPE................", b"SGC1xxxx", _hdr(1, 1, 1, 7), _hdr(0, 1, 1, 0),
             _hdr(2, 2, 1, 0) + b"\0" * 8, _hdr(1, 1, 1, 0) + b"\0" * 8, _hdr(1, 2, 1, 1) + b"\0" * 16]
    for data in cases:
        _bytes(p, data)
        try:
            want = ("ok", oracle.ref_load_tensor(p, f64=data[16:20] == b"\x01\0\0\0"))
        except oracle.OracleError as e:
            want = ("err", e.code, getattr(e, "offset", None))
        try:
            got = ("ok", sc.load_tensor(p).numpy())
        except sc.ParseError as e:
            got = ("err", 6, e.byte_offset)
        except sc.IoError:
            got = ("err", 5, None)
        if want[0] == "ok":
            assert got[0] == "ok"
            np.testing.assert_array_equal(got[1], want[1])
        else:
            assert got[:2] == want[:2] and (want[1] != 6 or got[2] == want[2]), data


def test_non_finite_payload_is_a_contract_error(tmp_path):
    """reference load_tensor builds its result through Tensor::from_data, which
    throws ContractError("tensor data contains a non-finite element")
    (tensor.hpp:87-88); the loaders here do the same, the batch loader too."""
    import struct
    cases = [(_hdr(1, 2, 1, 0) + struct.pack("<ff", 1.0, float("nan")), False),
             (_hdr(2, 1, 1, 0) + struct.pack("<ff", float("-inf"), 0.5), False),
             (_hdr(1, 1, 2, 1) + struct.pack("<dd", float("inf"), 2.0), True)]
    for i, (data, f64) in enumerate(cases):
        p = str(tmp_path / f"nf{i}.sgc")
        _bytes(p, data)
        with pytest.raises(sc.ContractError, match="non-finite"):
            sc.load_tensor(p)
        with pytest.raises(sc.ContractError, match="non-finite"):
            sc.load_tensor_batch([p])
        if oracle.ref_available():
            with pytest.raises(oracle.OracleError) as e:
                oracle.ref_load_tensor(p, f64=f64)
            assert e.value.code == 2 and "non-finite" in str(e.value)


def test_batch_loader_host(tmp_path):
    rng = np.random.default_rng(2)
    imgs = [rng.standard_normal((4, 4, 3)).astype(np.float32) for _ in range(5)]
    paths = []
    for i, a in enumerate(imgs):
        paths.append(str(tmp_path / f"{i}.sgc"))
        sc.save_tensor(torch.from_numpy(a), paths[-1])
    b = sc.load_tensor_batch(paths)
    np.testing.assert_array_equal(b.numpy(), np.stack(imgs))
    sc.save_tensor(torch.zeros((4, 5, 3)), paths[2])
    with pytest.raises(sc.ContractError):
        sc.load_tensor_batch(paths)


@pytest.mark.gpu
def test_batch_loader_uploads_and_feeds_the_fused_layer(tmp_path):
    """Files -> pinned staging -> device batch -> fused layer, checked against the oracle."""
    rng = np.random.default_rng(3)
    imgs = [rng.uniform(-1, 1, (16, 16, 64)).astype(np.float32) for _ in range(6)]
    paths = []
    for i, a in enumerate(imgs):
        paths.append(str(tmp_path / f"{i}.sgc"))
        sc.save_tensor(torch.from_numpy(a), paths[-1])
    xb = sc.load_tensor_batch(paths, device="cuda")
    assert xb.is_cuda and tuple(xb.shape) == (6, 16, 16, 64)
    k = (rng.standard_normal((3, 3, 64, 32)) * 0.05).astype(np.float32)
    y = sc.transpose_conv_fused(xb, torch.from_numpy(k).cuda(), 0).cpu().numpy()
    want = oracle.tconv_fused(np.stack(imgs), k, 0)
    err = np.abs(y - want) / np.maximum(np.maximum(np.abs(y), np.abs(want)), 1.0)
    assert err.max() <= 1e-5
    out = str(tmp_path / "y0.sgc")
    sc.save_tensor(torch.from_numpy(y[0]), out)
    np.testing.assert_array_equal(sc.load_tensor(out).numpy(), y[0])

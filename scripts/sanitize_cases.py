"""One small problem per kernel family, for compute-sanitizer (memcheck /
synccheck / racecheck): python scripts/sanitize_cases.py [family ...].
Each case asserts the kernel path it expects, so the sanitizer run covers
every family the dispatcher has.  Exit 0 when every case ran."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2209_03704_b200 import segconv as sc  # noqa: E402
from paper_2209_03704_b200 import stack as st  # noqa: E402


def t(a, dt=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)


rng = np.random.default_rng(3)


def fwd(b, n, cin, cout, k, p, dt, math, path, act=None):
    x = rng.standard_normal((b, n, n, cin)).astype(np.float32)
    w = (rng.standard_normal((k, k, cin, cout)) * 0.05).astype(np.float32)
    y = sc.transpose_conv_fused(t(x, dt), t(w, dt), p, math=math, activation=act)
    torch.cuda.synchronize()
    assert sc.last_path() == path, (sc.last_path(), path)
    return y


CASES = {
    "fold-ts": lambda: fwd(1, 64, 64, 32, 3, 0, torch.float32, "auto", "tc-fold-ts"),
    "ring": lambda: fwd(1, 128, 64, 3, 5, 0, torch.float32, "auto", "tc-ring", "tanh"),
    "fold": lambda: fwd(2, 20, 64, 8, 3, 0, torch.float32, "auto", "tc-fold"),
    "fold-bf16": lambda: fwd(2, 20, 64, 8, 3, 0, torch.bfloat16, "auto", "tc-fold"),
    "pair": lambda: fwd(4, 8, 128, 128, 4, 0, torch.bfloat16, "auto", "tc-pair", "relu"),
    "pair-split": lambda: fwd(2, 8, 128, 64, 4, 0, torch.float32, "auto", "tc-pair"),
    "pair-tf32": lambda: fwd(2, 8, 128, 64, 4, 0, torch.float32, "tf32", "tc-pair"),
    "pair-allq": lambda: fwd(1, 64, 128, 64, 4, 2, torch.bfloat16, "auto", "tc-pair"),
    "tile": lambda: fwd(8, 11, 128, 3, 3, 0, torch.bfloat16, "auto", "tc-tile", "tanh"),
    "halo": lambda: fwd(2, 6, 32, 48, 3, 2, torch.float32, "f16x3", "tc-halo"),
    "simt": lambda: fwd(1, 16, 8, 8, 3, 1, torch.float32, "ffma", "simt-tiled"),
    "exact": lambda: fwd(1, 6, 3, 2, 3, 1, torch.float32, "exact", "simt-exact"),
}


def backward_cases():
    x = rng.integers(-2, 3, (2, 6, 6, 128)).astype(np.float32)
    k = rng.integers(-2, 3, (4, 4, 128, 128)).astype(np.float32)
    gy = rng.integers(-2, 3, (2, 12, 12, 128)).astype(np.float32)
    sc.transpose_conv_fused_backward(t(x, torch.bfloat16), t(k, torch.bfloat16), 2, t(gy, torch.bfloat16))
    torch.cuda.synchronize()
    assert sc.last_path() == "bwd:tc-pair+tc-pair", sc.last_path()
    x = rng.uniform(-1, 1, (1, 64, 64, 64)).astype(np.float32)
    k = rng.uniform(-1, 1, (5, 5, 64, 3)).astype(np.float32)
    gy = rng.uniform(-1, 1, (1, 123, 123, 3)).astype(np.float32)
    sc.transpose_conv_fused_backward(t(x), t(k), 0, t(gy))
    torch.cuda.synchronize()
    assert sc.last_path() == "bwd:simt-narrow+simt-narrow", sc.last_path()


def conv_valid_case():
    x = rng.standard_normal((2, 10, 10, 64)).astype(np.float32)
    k = (rng.standard_normal((3, 3, 64, 64)) * 0.05).astype(np.float32)
    sc.conv2d_valid(t(x, torch.bfloat16), t(k, torch.bfloat16))
    torch.cuda.synchronize()
    assert sc.last_path() == "tc-pair", sc.last_path()
    sc.transpose_conv_naive(t(x[:, :5, :5, :8]), t(k[:, :, :8, :4]), 1, math="exact")
    torch.cuda.synchronize()


def stack_case():
    specs = st.c5_layers()
    ks = [torch.from_numpy((rng.standard_normal((s.k, s.k, s.cin, s.cout)) * 0.02).astype(np.float32))
          for s in specs]
    m = st.MultiGPUStack(specs, ks, 8, n_gpus=1)
    m.forward(torch.from_numpy(rng.standard_normal((8, 4, 4, 1024)).astype(np.float32)).bfloat16())
    m.close()
    g = st.GeneratorStack(specs, [k.cuda() for k in ks], 8)
    g.capture()
    g.forward()
    torch.cuda.synchronize()


CASES["backward"] = backward_cases
CASES["conv-valid"] = conv_valid_case
CASES["stack"] = stack_case

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        print("ok", n, flush=True)

"""Quick parity check of the pixel-scatter ring kernel (C4 shape family) against the C oracle."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2209_03704_b200 import segconv as sc

def check(b, n, cin, act, bias=False):
    rng = np.random.default_rng(b * 13 + n)
    x = rng.uniform(-1, 1, (b, n, n, cin)).astype(np.float32)
    w = (rng.standard_normal((5, 5, cin, 3)) * 0.02).astype(np.float32)
    bb = rng.uniform(-0.1, 0.1, 3).astype(np.float32) if bias else None
    g = sc.tconv_geometry(n, 5, 5, 0)
    sks = sc.segregate(torch.from_numpy(w).cuda(), 0, math="f16x3")
    y = sc.transpose_conv_fused(torch.from_numpy(x).cuda(), sks, g, activation=act,
                                bias=torch.from_numpy(bb).cuda() if bias else None)
    torch.cuda.synchronize()
    want = oracle.tconv_fused(x, w, 0)
    if bias: want = want + bb
    if act == "tanh": want = np.tanh(want)
    got = y.cpu().numpy()
    err = np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), 1.0)
    i = np.unravel_index(np.argmax(err), err.shape)
    print(f"b{b} n{n} cin{cin} act={act}: max scaled err {err.max():.2e} at {i} got {got[i]} want {want[i]}", flush=True)
    return err.max()

errs = [check(1, 128, 64, None), check(2, 128, 64, "tanh", True), check(3, 256, 32, None), check(1, 256, 64, "tanh")]
print("RING", "OK" if max(errs) <= 1e-5 else "FAIL")

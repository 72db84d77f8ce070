"""Quick parity check of the small-image pixel-scatter kernel (C5 layer d family) against the C oracle."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2209_03704_b200 import segconv as sc

def check(b, n, cin, act, out_dtype=torch.float32):
    rng = np.random.default_rng(b * 17 + n)
    x = oracle.bf16_round(rng.standard_normal((b, n, n, cin)).astype(np.float32))
    w = oracle.bf16_round((rng.standard_normal((3, 3, cin, 3)) * 0.02).astype(np.float32))
    g = sc.tconv_geometry(n, 3, 3, 0)
    sks = sc.segregate(torch.from_numpy(w).cuda().to(torch.bfloat16), 0, math="bf16")
    y = sc.transpose_conv_fused(torch.from_numpy(x).cuda().to(torch.bfloat16), sks, g,
                                activation=act, out_dtype=out_dtype)
    torch.cuda.synchronize()
    want = oracle.tconv_fused(x, w, 0)
    if act == "tanh": want = np.tanh(want)
    got = y.float().cpu().numpy()
    err = np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), 1.0)
    print(f"b{b} n{n} cin{cin} act={act} {out_dtype}: max scaled err {err.max():.2e}", flush=True)
    return err.max() if out_dtype == torch.float32 else err.max() / 1e3

errs = [check(4, 11, 128, "tanh"), check(3, 7, 64, None), check(5, 16, 128, "tanh", torch.bfloat16),
        check(2, 30, 192, None)]
print("TILE", "OK" if max(errs) <= 1e-5 else "FAIL")

"""Quick parity check of the CTA-pair bf16 kernel against the C oracle (bf16-rounded inputs)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2209_03704_b200 import segconv as sc

def check(b, n, cin, cout, k, p=0, act=None):
    rng = np.random.default_rng(b * 7 + n)
    x = oracle.bf16_round(rng.standard_normal((b, n, n, cin)).astype(np.float32))
    w = oracle.bf16_round((rng.standard_normal((k, k, cin, cout)) * 0.02).astype(np.float32))
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    wt = torch.from_numpy(w).cuda().to(torch.bfloat16)
    g = sc.tconv_geometry(n, k, k, p)
    sks = sc.segregate(wt, p, math="bf16")
    y = sc.transpose_conv_fused(xt, sks, g, activation=act, out_dtype=torch.float32)
    torch.cuda.synchronize()
    want = oracle.tconv_fused(x[:2], w, p)
    if act == "relu": want = np.maximum(want, 0)
    got = y[:2].cpu().numpy()
    err = np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), 1.0)
    print(f"b{b} n{n} {cin}->{cout} k{k} layout={sks.layout}: max scaled err {err.max():.2e}", flush=True)
    return err.max()

errs = [check(4, 16, 512, 256, 4), check(3, 4, 1024, 512, 3, act="relu"), check(2, 7, 256, 128, 3),
        check(5, 5, 512, 256, 3), check(2, 9, 64, 96, 4)]
print("WIDE", "OK" if max(errs) <= 1e-3 else "FAIL")  # bf16 tensor-core bar is 1e-2

"""Timeline of the tc-tile kernel (SEGCONV_TC_TRACE=1) for C5 layer d: kernel
entry (ev6), setup done (ev8), per tile producer start (ev0), MMA start (ev2),
epilogue start / end (ev4 / ev5), exit (ev7); L2 flushed before the traced call
unless NOFLUSH=1.  python scripts/trace_tile.py [B N CIN]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2209_03704_b200 import _capi as A  # noqa: E402
from paper_2209_03704_b200 import segconv as sc  # noqa: E402

b, n, cin = (int(v) for v in (sys.argv[1:4] or (1024, 11, 128)))
x = torch.randn((b, n, n, cin), device="cuda").bfloat16()
w = (torch.randn((3, 3, cin, 3), device="cuda") * 0.02).bfloat16()
g = sc.tconv_geometry(n, 3, 3, 0)
sks = sc.segregate(w, 0)
y = torch.empty((b, g.out_h, g.out_w, 3), device="cuda", dtype=torch.bfloat16)
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    sc.transpose_conv_fused(x, sks, g, out=y)
torch.cuda.synchronize()
if not os.environ.get("NOFLUSH"):
    flush.fill_(1)
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
sc.transpose_conv_fused(x, sks, g, out=y)
e.record()
torch.cuda.synchronize()
print("event time", round(a.elapsed_time(e) * 1000, 2), "us", sc.last_path())
buf = np.zeros(160 * 16 * 64, dtype=np.uint64)
A.lib().segconv_debug_trace(buf.ctypes.data_as(C.c_void_p), buf.nbytes)
tr = buf.reshape(160, 16, 64).astype(np.int64)
t0 = tr[:, 6, 0][tr[:, 6, 0] > 0].min()
us = lambda v: (v - t0) / 1000  # noqa: E731
ent, setup, ex = tr[:, 6, 0], tr[:, 8, 0], tr[:, 7, 0]
ok = ent > 0
print(f"entry  min {us(ent[ok].min()):.2f} max {us(ent[ok].max()):.2f}")
print(f"setup  min {us(setup[ok].min()):.2f} max {us(setup[ok].max()):.2f}")
print(f"exit   min {us(ex[ok].min()):.2f} max {us(ex[ok].max()):.2f}")
for cta in (0, 1, 100, 147, 148, 159):
    print("CTA", cta, f"entry {us(ent[cta]):.2f} setup {us(setup[cta]):.2f} exit {us(ex[cta]):.2f}")
    for u in range(8):
        row = tr[cta, :6, u]
        if not row.any():
            break
        print(f"  tile {u}: " + " ".join(f"ev{q}={us(v):6.2f}" for q, v in enumerate(row) if v))

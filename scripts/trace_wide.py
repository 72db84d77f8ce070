"""Per-unit timeline of the CTA-pair kernel (SEGCONV_TC_TRACE=1): producer
done (ev 0), MMA start/end (2/3), epilogue start (4), for CTA 0.
python scripts/trace_wide.py B N CIN COUT K P"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2209_03704_b200 import _capi as A  # noqa: E402
from paper_2209_03704_b200 import segconv as sc  # noqa: E402

b, n, cin, cout, k, p = (int(v) for v in sys.argv[1:7])
x = torch.randn((b, n, n, cin), device="cuda").bfloat16()
w = (torch.randn((k, k, cin, cout), device="cuda") * 0.02).bfloat16()
g = sc.tconv_geometry(n, k, k, p)
sks = sc.segregate(w, p)
for _ in range(3):
    sc.transpose_conv_fused(x, sks, g)
torch.cuda.synchronize()
sc.transpose_conv_fused(x, sks, g)
torch.cuda.synchronize()
buf = np.zeros(160 * 16 * 64, dtype=np.uint64)
A.lib().segconv_debug_trace(buf.ctypes.data_as(C.c_void_p), buf.nbytes)
tr = buf.reshape(160, 16, 64).astype(np.int64)
t0 = tr[tr > 0].min()
import os
ctas = [int(c) for c in os.environ.get("TRACE_CTAS", "0,2").split(",")]
for cta in ctas:
    print("CTA", cta, sc.last_path())
    for u in range(20):
        row = tr[cta, :6, u]
        if not row.any():
            break
        print(f"  unit {u}: " + " ".join(f"ev{e}={(v - t0) / 1000:7.2f}" for e, v in enumerate(row) if v))

# per stage (im2col path, CTA 0): 10 A producer slot free, 11 B producer slot free, 6 MMA saw data, 8 MMA committed
if os.environ.get("TRACE_STAGES"):
    print("stage: A slot free / B slot free / MMA data ready / committed (us)")
    for g in range(64):
        row = [tr[0, e, g] for e in (10, 11, 6, 8)]
        if not row[2]:
            break
        print("  g=%2d " % g + " ".join(f"{(v - t0) / 1000:7.2f}" if v else "   -   " for v in row))

# start / end of every CTA (unit 0 MMA start, last epilogue end): a second wave
# of clusters shows as CTAs that start when others finish
if os.environ.get("TRACE_WAVES"):
    st, en = [], []
    for cta in range(160):
        row = tr[cta]
        if not row[2].any():
            continue
        st.append((row[2][row[2] > 0].min() - t0) / 1000)
        en.append((row[5][row[5] > 0].max() - t0) / 1000 if row[5].any() else 0)
    st, en = np.array(st), np.array(en)
    print(f"CTAs with events {len(st)}; start min {st.min():.2f} max {st.max():.2f}; end min {en.min():.2f} max {en.max():.2f}")
    print("starts sorted:", np.round(np.sort(st), 2)[-20:])

# CTA lifetimes (ev12 = setup done, ev13 = exit), all traced CTAs
st, ex = tr[:, 12, 0], tr[:, 13, 0]
ok = ex > 0
if ok.any():
    exs = np.sort((ex[ok] - t0) / 1000)
    print(f"setup done: min {(st[ok].min() - t0) / 1000:.2f} max {(st[ok].max() - t0) / 1000:.2f} us")
    print("exit percentiles (us): " + " ".join(f"p{q}={np.percentile(exs, q):.2f}" for q in (0, 10, 25, 50, 75, 90, 100)))
    nun = [(tr[c, 5, :] > 0).sum() for c in range(160) if ex[c] > 0]
    print("units per CTA:", sorted(set(nun)), "mean busy fraction:",
          round(float(np.mean(exs) / exs.max()), 3))

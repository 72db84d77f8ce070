"""Per-unit pipeline timeline of the tcgen05 kernel (diagnostics).
Run with SEGCONV_TC_TRACE=1:  python scripts/trace_tc.py C2"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2209_03704_b200 import _capi as A  # noqa: E402
from paper_2209_03704_b200 import segconv as sc  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
prob = bench.Layer(cfg, 0, torch, sc, torch.device("cuda", 0), 1)
for _ in range(3):
    prob.step()
torch.cuda.synchronize()
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
if os.environ.get("TRACE_FLUSH", "1") == "1":  # cold L2, as in bench.py
    flush.fill_(1)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
prob.step()
b.record()
torch.cuda.synchronize()
print("kernel ms", a.elapsed_time(b))
buf = np.zeros(160 * 16 * 64, dtype=np.uint64)
n = A.lib().segconv_debug_trace(buf.ctypes.data_as(C.c_void_p), buf.nbytes)
tr = buf.reshape(160, 16, 64).astype(np.int64)
names = ["A-tma", "conv", "mma0", "mma1", "epi0", "epi1", "wland", "wtmem", "epiB1", "entry", "prolog", "exit"]
t0 = tr[:, :12][tr[:, :12] > 0].min()
for cta in range(2):
    print(f"CTA {cta}")
    for u in range(64):
        row = tr[cta, :12, u]
        if not row.any():
            break
        print(f"  unit {u}: " + "  ".join(f"{nm}={(v - t0) / 1000:7.2f}us" if v else f"{nm}=   -   "
                                          for nm, v in zip(names, row)))

# all-CTA summary: first A-TMA and last epilogue-done per CTA
starts, ends, nunits = [], [], []
for cta in range(160):
    row = tr[cta]
    if not row.any():
        continue
    starts.append(row[row > 0].min())
    ends.append(row[5][row[5] > 0].max() if (row[5] > 0).any() else 0)
    nunits.append(int((row[5] > 0).sum()))
starts, ends = np.array(starts), np.array(ends)
print(f"CTAs {len(starts)}: start spread {(starts.max()-starts.min())/1000:.2f}us, "
      f"end min {(ends.min()-t0)/1000:.2f}us max {(ends.max()-t0)/1000:.2f}us, units/CTA {min(nunits)}-{max(nunits)}")
slow = np.argsort(ends)[-3:]
for c in slow:
    print("  slowest CTA", c, f"end {(ends[c]-t0)/1000:.2f}us start {(starts[c]-t0)/1000:.2f}us units {nunits[c]}")

ent = tr[:, 9, 0]
ext = tr[:, 11, 0]
ok = (ent > 0) & (ext > 0)
if ok.any():
    print(f"kernel span (entry..exit over CTAs): first entry {(ent[ok].min()-t0)/1000:.2f}us, "
          f"last entry {(ent[ok].max()-t0)/1000:.2f}us, last exit {(ext[ok].max()-t0)/1000:.2f}us, "
          f"prologue max {((tr[:,10,0]-ent)[ok]).max()/1000:.2f}us")

ck = tr[:, 13, 0] - tr[:, 12, 0]
ns = tr[:, 11, 0] - tr[:, 9, 0]
okc = ok & (ck > 0) & (ns > 0)
if okc.any():
    f = ck[okc] / ns[okc]
    print(f"SM clock during the kernel: {f.mean():.3f} GHz (min {f.min():.3f}, max {f.max():.3f})")

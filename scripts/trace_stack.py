"""Timeline of the C5 stack graph (SEGCONV_TC_TRACE=2: one trace slot per
launch): per layer, kernel entry of its first / last CTA, setup done, first
activation load (after griddepcontrol.wait), last CTA exit -- where the step's
time between the layers goes.  L2 flushed before the traced replay.
python scripts/trace_stack.py [batch]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
assert os.environ.get("SEGCONV_TC_TRACE") == "2", "run with SEGCONV_TC_TRACE=2"
import bench  # noqa: E402
from paper_2209_03704_b200 import _capi as A  # noqa: E402
from paper_2209_03704_b200 import segconv as sc  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = dict(bench.CONFIGS["C5"])
prob = bench.Stack(cfg, 0, 1, torch, sc, torch.device("cuda"), batch=batch, with_capi=False)
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    prob.step()
torch.cuda.synchronize()
flush.fill_(1)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
prob.step()
b.record()
torch.cuda.synchronize()
print(f"graph step {a.elapsed_time(b) * 1000:.1f} us (events)")
SLOT = 160 * 16 * 64
buf = np.zeros(8 * SLOT, dtype=np.uint64)
n = A.lib().segconv_debug_trace(buf.ctypes.data_as(C.c_void_p), buf.nbytes)
tr = buf[: n // 8].reshape(-1, 160, 16, 64).astype(np.int64)
# the last replay's four launches: the slots holding the latest stamps
last = sorted(range(tr.shape[0]), key=lambda s: tr[s].max())[-4:]
last.sort(key=lambda s: tr[s][tr[s] > 0].min())
t0 = min(tr[s][tr[s] > 0].min() for s in last)
us = lambda v: (v - t0) / 1000.0  # noqa: E731
prev_exit = None
for name, s in zip("abcd", last):
    t = tr[s]
    if t[:, 13, 0].any():  # pair kernel: 14 entry, 12 setup, 10 first A stage, 13 exit
        ent, setup, first, ex = t[:, 14, 0], t[:, 12, 0], t[:, 10, 0], t[:, 13, 0]
    else:  # tile kernel: 6 entry, 8 setup, 0 first tile issued, 7 exit
        ent, setup, first, ex = t[:, 6, 0], t[:, 8, 0], t[:, 0, 0], t[:, 7, 0]
    ok = ent > 0
    f = first[first > 0]
    line = (f"layer {name}: entry {us(ent[ok].min()):7.2f}..{us(ent[ok].max()):7.2f}  setup<= {us(setup[ok].max()):7.2f}"
            f"  first load {us(f.min()):7.2f}..{us(f.max()):7.2f}  exit {us(ex[ok].min()):7.2f}..{us(ex[ok].max()):7.2f}")
    if prev_exit is not None:
        line += f"  gap(prev last exit -> first load) {us(f.min()) - us(prev_exit):5.2f}"
    print(line)
    if t[:, 13, 0].any():  # pair-kernel prologue, CTA 0 and the latest-entering CTA
        for c in (0, 1, int(np.argmax(np.where(ok, ent, 0)))):
            print(f"   CTA {c}: entry {us(ent[c]):.2f} barriers {us(t[c, 15, 1]) if t[c, 15, 1] else float('nan'):.2f}"
                  f" tmem {us(t[c, 15, 0]) if t[c, 15, 0] else float('nan'):.2f} sync {us(t[c, 15, 2]):.2f}"
                  f" cluster {us(t[c, 15, 3]):.2f} setup {us(setup[c]):.2f} first load {us(first[c]) if first[c] else float('nan'):.2f}")
    prev_exit = ex[ok].max()

"""Diagnostics: one layer's step time after three L2 states -- a 256 MiB
write (bench.py's flush: L2 left full of dirty lines that the timed kernel
must write back as it allocates), a 256 MiB read (cold but clean L2) and no
flush (inputs warm).  python scripts/flush_modes.py [config]"""
import statistics, sys, torch
sys.path.insert(0, ".")
import bench
from paper_2209_03704_b200 import segconv as sc
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = bench.CONFIGS[name]
prob = bench.Layer(cfg, 0, torch, sc, torch.device("cuda", 0), 1)
buf = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
buf2 = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
buf2.fill_(3)
for _ in range(3): prob.step()
torch.cuda.synchronize()
def timeit(pre):
    ts = []
    for i in range(40):
        pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); prob.step(); b.record(); b.synchronize()
        if i >= 5: ts.append(a.elapsed_time(b) * 1000)
    return statistics.median(ts)
print(name, "write-flush %.2f us" % timeit(lambda: buf.fill_(1)))
print(name, "write-flush + clean read %.2f us" % timeit(lambda: (buf.fill_(1), buf2.sum())))
print(name, "read-flush %.2f us" % timeit(lambda: buf2.sum()))
print(name, "no flush %.2f us" % timeit(lambda: None))

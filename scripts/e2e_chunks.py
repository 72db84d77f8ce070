import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2209_03704_b200 import segconv as sc
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.uniform(-1, 1, (16, 64, 64, 64)).astype(np.float32)).pin_memory()
k = torch.from_numpy((rng.standard_normal((3, 3, 64, 32)) * 0.059).astype(np.float32)).cuda()
g = sc.tconv_geometry(64, 3, 3, 0)
sks = sc.segregate(k, 0)
yh = torch.empty((16, 125, 125, 32), pin_memory=True)
xd = torch.empty(x.shape, device="cuda"); yd = torch.empty(yh.shape, device="cuda")
s = torch.cuda.current_stream()
for ch in [1, 2, 4, 8, 16]:
    for _ in range(3):
        sc.transpose_conv_fused(x, sks, g, out=yh, staging=(xd, yd), chunks=ch, sync=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        sc.transpose_conv_fused(x, sks, g, out=yh, staging=(xd, yd), chunks=ch, sync=False)
    b.record(); torch.cuda.synchronize()
    print("chunks", ch, "ms/step", a.elapsed_time(b) / 20)
# pure copies for reference
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): xd.copy_(x, non_blocking=True)
b.record(); torch.cuda.synchronize(); print("H2D 16.8MB ms", a.elapsed_time(b) / 20)
a.record()
for _ in range(20): yh.copy_(yd, non_blocking=True)
b.record(); torch.cuda.synchronize(); print("D2H 32MB ms", a.elapsed_time(b) / 20)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
a.record()
for _ in range(20):
    with torch.cuda.stream(s1): xd.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2): yh.copy_(yd, non_blocking=True)
s.wait_stream(s1); s.wait_stream(s2)
b.record(); torch.cuda.synchronize(); print("both concurrently ms", a.elapsed_time(b) / 20)

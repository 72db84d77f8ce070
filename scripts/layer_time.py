"""Times single layers (bf16 or fp32) through transpose_conv_fused: python
scripts/layer_time.py B N CIN COUT K P [dtype]; LAYER_MATH=tf32|f16x3|bf16|ffma picks
the math (default auto); NOFLUSH=1 skips the L2 flush; prints path and us per call."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2209_03704_b200 import segconv as sc  # noqa: E402

b, n, cin, cout, k, p = (int(v) for v in sys.argv[1:7])
dt = torch.float32 if (len(sys.argv) > 7 and sys.argv[7] == "f32") else torch.bfloat16
x = torch.randn((b, n, n, cin), device="cuda").to(dt)
w = (torch.randn((k, k, cin, cout), device="cuda") * 0.02).to(dt)
g = sc.tconv_geometry(n, k, k, p)
import os  # noqa: E402
sks = sc.segregate(w, p, math=os.environ.get("LAYER_MATH", "auto"))
y = torch.empty((b, g.out_h, g.out_w, cout), device="cuda", dtype=dt)
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    sc.transpose_conv_fused(x, sks, g, out=y)
ts = []
for _ in range(20):
    if not os.environ.get("NOFLUSH"):
        flush.fill_(1)
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sc.transpose_conv_fused(x, sks, g, out=y)
    e.record()
    e.synchronize()
    ts.append(a.elapsed_time(e) * 1000)
print(sys.argv[1:], sc.last_path(), round(statistics.median(ts), 2), "us")

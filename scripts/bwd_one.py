"""One backward part on one config, a few reps (for ncu launch lists)."""
import sys

import torch

sys.path.insert(0, ".")
from bench import CONFIGS  # noqa: E402
from paper_2209_03704_b200 import segconv as sc  # noqa: E402

name, part = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
c = CONFIGS[name]
dt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
b, n, cin, cout, k, p = c["batch"], c["n"], c["cin"], c["cout"], c["k"], c["p"]
g = sc.tconv_geometry(n, k, k, p)
x = torch.randn((b, n, n, cin), device="cuda").to(dt)
kk = (torch.randn((k, k, cin, cout), device="cuda") * 0.02).to(dt)
gy = torch.randn((b, g.out_h, g.out_w, cout), device="cuda").to(dt)
for _ in range(reps):
    sc.transpose_conv_fused_backward(x, kk, p, gy, input_grad=part == "input", kernel_grad=part == "kernel")
torch.cuda.synchronize()
print(sc.last_path())

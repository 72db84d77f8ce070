"""Diagnostics: one C2-shaped kernel gradient (fp32, FFMA) for an ncu launch list."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2209_03704_b200 import segconv as sc  # noqa: E402
x = torch.rand((16, 64, 64, 64), device="cuda") * 2 - 1
k = torch.randn((3, 3, 64, 32), device="cuda") * 0.059
g = sc.tconv_geometry(64, 3, 3, 0)
gy = torch.rand((16, g.out_h, g.out_w, 32), device="cuda") * 2 - 1
for _ in range(3):
    sc.transpose_conv_fused_backward(x, k, 0, gy, input_grad=False, kernel_grad=True)
torch.cuda.synchronize()
print(sc.last_path())

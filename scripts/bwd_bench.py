"""Times the backward kernels (input gradient, kernel gradient) on the BASELINE
layer shapes with CUDA events; prints one JSON line per (config, part)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from bench import CONFIGS  # noqa: E402
from paper_2209_03704_b200 import segconv as sc  # noqa: E402


def main():
    names = sys.argv[1:] or ["C2", "C3", "C4", "C5a", "C5b", "C5c", "C5d"]
    for name in names:
        c = CONFIGS[name]
        dt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
        b, n, cin, cout, k, p = c["batch"], c["n"], c["cin"], c["cout"], c["k"], c["p"]
        g = sc.tconv_geometry(n, k, k, p)
        x = torch.randn((b, n, n, cin), device="cuda").to(dt)
        kk = (torch.randn((k, k, cin, cout), device="cuda") * 0.02).to(dt)
        gy = torch.randn((b, g.out_h, g.out_w, cout), device="cuda").to(dt)
        macs = b * n * n * cin * cout * k * k  # dense (every tap reaches every pixel, minus borders)
        for part in ("input", "kernel", "both"):
            kw = dict(input_grad=part != "kernel", kernel_grad=part != "input")
            for _ in range(3):
                sc.transpose_conv_fused_backward(x, kk, p, gy, **kw)
            torch.cuda.synchronize()
            path = sc.last_path()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            e0.record()
            for _ in range(reps):
                sc.transpose_conv_fused_backward(x, kk, p, gy, **kw)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1000 / reps
            m = macs * (2 if part == "both" else 1)
            print(json.dumps({"config": name, "part": part, "path": path, "us": round(us, 2),
                              "tflops": round(2 * m / us / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()

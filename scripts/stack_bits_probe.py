import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2209_03704_b200 import stack as st
specs = st.c5_layers()
rng = np.random.default_rng(57)
ks = [torch.from_numpy(rng.standard_normal((s.k, s.k, s.cin, s.cout), dtype=np.float32) * 0.02) for s in specs]
x = torch.from_numpy(rng.standard_normal((1024, 4, 4, 1024), dtype=np.float32)).bfloat16()
for b in (1024, 256, 128):
    ref = st.GeneratorStack(specs, [k.cuda() for k in ks], 1024).forward(x.cuda()).cpu()[:b]
    g2 = st.GeneratorStack(specs, [k.cuda() for k in ks], b).forward(x[:b].cuda()).cpu()
    d = (g2.float() - ref.float()).abs()
    print("graph", b, "vs 1024: differing", int((d > 0).sum()), "max", float(d.max()))
ms = st.MultiGPUStack(specs, ks, 1024, n_gpus=1)
y = ms.forward(x.pin_memory())
ref = st.GeneratorStack(specs, [k.cuda() for k in ks], 1024).forward(x.cuda()).cpu()
d = (y.float() - ref.float()).abs()
print("capi 1024 vs graph 1024: differing", int((d > 0).sum()), "of", d.numel(), "max", float(d.max()))

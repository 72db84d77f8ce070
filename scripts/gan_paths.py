import sys, torch
sys.path.insert(0, ".")
from paper_2209_03704_b200 import segconv as sc, stack as st
for m in st.GAN_MODELS:
    for s in st.gan_layers(m):
        x = torch.randn((8, s.n_in, s.n_in, s.cin), device="cuda").bfloat16()
        k = (torch.randn((4, 4, s.cin, s.cout), device="cuda") * 0.02).bfloat16()
        sc.transpose_conv_fused(x, k, 2)
        print(m, s.n_in, s.cin, s.cout, sc.last_path())

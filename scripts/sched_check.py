import os, sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2405_12591_b200.attention import DecodeKvCache
units, T = 512, 4096
c = DecodeKvCache(layers=1, units=units, g=1, bits=4, tc=True)
k = torch.randn((units, T, 128), device="cuda").half()
c.prefill(0, k, k)
q = torch.randn((units, 1, 128), device="cuda").half()
out = torch.empty_like(q)
sched = c._layers[0].keep[3] if c._layers[0].args else None
c.attend(0, q, out)
torch.cuda.synchronize()
print("sched after attend", c._layers[0].keep[3].cpu().tolist())
for i in range(3):
    c.launch(0, q, out, phases=1); torch.cuda.synchronize()
    print("sched after split", c._layers[0].keep[3].cpu().tolist())

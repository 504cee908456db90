# measurement only: C2 step with and without the prepare kernel (W images from the first launch)
import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2405_12591_b200.attention import DecodeKvCache
L, U, T = 32, 512, 4096
cache = DecodeKvCache(layers=L, units=U, g=1, bits=4)
g = torch.Generator(device="cuda"); g.manual_seed(0)
k = torch.randn((U, T, 128), generator=g, device="cuda").half()
for l in range(L):
    cache.prefill(l, k, k)
q = torch.randn((L, U, 1, 128), generator=g, device="cuda").half()
out = torch.empty_like(q)
for l in range(L):
    cache.attend(l, q[l], out[l])
torch.cuda.synchronize()
def run(phases, n=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        for l in range(L): cache.launch(l, q[l], out[l], phases=phases)
    e0.record()
    for _ in range(n):
        for l in range(L): cache.launch(l, q[l], out[l], phases=phases)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
print("all phases %.3f ms/step, without prepare %.3f, split only %.3f" % (run(7), run(3), run(1)))

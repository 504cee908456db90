import sys, os, torch, json
sys.path.insert(0, os.getcwd())
from paper_2405_12591_b200.model import LLAMA2_7B, DecoQuantLM
from torch.profiler import profile, ProfilerActivity
lm = DecoQuantLM(LLAMA2_7B, 16); lm.prefill_random(4096)
tok = torch.zeros(16, dtype=torch.int64, device="cuda")
for _ in range(3): tok = lm.step(tok)
lm.capture()
for _ in range(3): tok = lm.replay(tok)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    for _ in range(5): tok = lm.replay(tok)
    torch.cuda.synchronize()
agg = {}
for e in p.events():
    if e.device_type.name == "CUDA":
        k = e.name[:90]; a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += e.device_time_total if hasattr(e,'device_time_total') else e.cuda_time_total
tot = sum(v[1] for v in agg.values())
print("total us/step", tot / 5, "kernels/step", sum(v[0] for v in agg.values()) / 5)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{v[1]/5:9.1f} us {v[0]/5:6.0f}x  {k}")

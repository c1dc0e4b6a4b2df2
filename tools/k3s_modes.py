"""dev->dev timing of the OPT-1.3B set (K3s tuning aid)."""
import sys, time
import torch
sys.path.insert(0, ".")
from bench import layer_shapes
from paper_2403_02775_b200 import native as N
shapes = layer_shapes("opt-1.3b")
g = torch.Generator(device="cuda").manual_seed(1)
Ws = [torch.randn(s, generator=g, device="cuda") * 0.02 for s in shapes]
cfg = N.Config()
N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()
torch.cuda.synchronize()
N.profile_enable(True)
t0 = time.perf_counter()
for _ in range(3):
    N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 3
prof = {"ms": N.profile_read("qrange")["ms"] + N.profile_read("qsort")["ms"]}
N.profile_enable(False)
print(f"dev->dev {dt*1e3:.1f} ms/call, qrange {prof['ms']/3:.1f} ms/call")

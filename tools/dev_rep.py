"""Repeated device-in/device-out calls on the OPT-1.3B set, one timing per call (dev aid)."""
import sys, time
import torch
sys.path.insert(0, ".")
from bench import layer_shapes
from paper_2403_02775_b200 import native as N
shapes = layer_shapes("opt-1.3b")
g = torch.Generator(device="cuda").manual_seed(1)
Ws = [torch.randn(s, generator=g, device="cuda") * 0.02 for s in shapes]
cfg = N.Config()
out = []
for i in range(12):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()
    torch.cuda.synchronize()
    out.append((time.perf_counter() - t0) * 1e3)
print(" ".join(f"{x:.1f}" for x in out))

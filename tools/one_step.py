"""One quantize_batch of a bench workload, device in/out, after one warm-up
call (for ncu launch lists: `ncu -k regex:^k_ ... python tools/one_step.py`;
the warm-up's launches come first, `--launch-skip` past them or split by
count)."""
import argparse
import sys
import torch
sys.path.insert(0, ".")
from bench import layer_shapes
from paper_2403_02775_b200 import native as N
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="opt-1.3b")
ap.add_argument("--warm", type=int, default=0)
ap.add_argument("--sigma", type=float, default=3.0)
a = ap.parse_args()
shapes = layer_shapes(a.workload)
g = torch.Generator(device="cuda").manual_seed(1)
Ws = [torch.randn(s, generator=g, device="cuda") * 0.02 for s in shapes]
cfg = N.Config(sigma_n=a.sigma)
for _ in range(a.warm + 1):
    N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()
torch.cuda.synchronize()
print("launches", N.kernel_launches())

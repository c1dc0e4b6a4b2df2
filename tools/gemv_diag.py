import sys, torch
sys.path.insert(0, ".")
from paper_2403_02775_b200 import native as N
from paper_2403_02775_b200.native import Config
r, c, B, dt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
W = torch.randn(r, c, device="cuda") * 0.02
b = N.quantize_batch([W], Config(sigma_n=1e4, steps=5), "outliers-only", out_mem=N.MEM_DEVICE)
torch.cuda.synchronize(); print("quantized", flush=True)
p = N.GemvPlan(b, 0)
torch.cuda.synchronize(); print("prepared", flush=True)
x = torch.randn(B, r, device="cuda").to(getattr(torch, dt))
y = p(x); torch.cuda.synchronize(); print("gemv ok", float(y.abs().max()), flush=True)

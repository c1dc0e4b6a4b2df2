import sys, torch
sys.path.insert(0, ".")
from paper_2403_02775_b200 import native as N
W = [torch.randn(2048, 2048, device="cuda") * 0.02 for _ in range(4)]
for _ in range(2):
    N.quantize_batch(W, N.Config(), out_mem=N.MEM_DEVICE).close()
torch.cuda.synchronize()

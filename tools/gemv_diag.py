"""GEMV smoke/diagnostic (development aid): one quantize + prepare + GEMV,
synchronizing after each step.  python tools/gemv_diag.py ROWS COLS BATCH XDTYPE [SIGMA_N] [OUTLIER_DTYPE]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2403_02775_b200 import native as N  # noqa: E402
from paper_2403_02775_b200.native import Config  # noqa: E402

r, c, B, dt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
sig = float(sys.argv[5]) if len(sys.argv) > 5 else 1e4
odt = sys.argv[6] if len(sys.argv) > 6 else "float32"
W = torch.randn(r, c, device="cuda") * 0.02
b = N.quantize_batch([W], Config(sigma_n=sig, steps=5), "outliers-only", out_mem=N.MEM_DEVICE)
torch.cuda.synchronize()
print("quantized, outliers", b[0].n_outliers, flush=True)
p = N.GemvPlan(b, 0, outlier_dtype=odt)
torch.cuda.synchronize()
print("prepared", flush=True)
x = torch.randn(B, r, device="cuda").to(getattr(torch, dt))
y = p(x)
torch.cuda.synchronize()
print("gemv ok", float(y.abs().max()), flush=True)

"""Numerics of the fused GEMV at the BLOOM-176B FFN shape (14336x53746, 1% outliers): K6 fused vs
the separate outlier pass vs dequantize + a torch fp32 matmul (dev check; the parity tests use
smaller shapes)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_02775_b200 import native as N  # noqa: E402
from paper_2403_02775_b200.native import Config  # noqa: E402

r, c = 14336, 53746
g = torch.Generator(device="cuda").manual_seed(5)
W = torch.randn(r, c, generator=g, device="cuda") * 0.02
b = N.quantize_batch([W], Config(sigma_n=2.5758), "outliers-only", out_mem=N.MEM_DEVICE)
del W
What = torch.empty(r, c, device="cuda")
b.dequantize_into(0, What)
os.environ["EZQ_GEMV_FUSED"] = "1"
pf = N.GemvPlan(b, 0)
os.environ["EZQ_GEMV_FUSED"] = "0"
ps = N.GemvPlan(b, 0)
for B in (1, 8, 16):
    for dt in (torch.bfloat16, torch.float32):
        x = torch.randn(B, r, generator=g, device="cuda").to(dt)
        yf, ys = pf(x), ps(x)
        ref = x.double().matmul(What.double()) if B == 1 else (x.float() @ What).double()
        sc = ref.abs().max().item()
        ef = (yf.double() - ref).abs().max().item() / sc
        es = (ys.double() - ref).abs().max().item() / sc
        print(f"B={B} {str(dt)[6:]}: fused rel err {ef:.2e}, separate {es:.2e}, fused==separate within {((yf - ys).abs().max().item() / sc):.2e}")
        assert ef <= 1e-3 and es <= 1e-3
print("ok")

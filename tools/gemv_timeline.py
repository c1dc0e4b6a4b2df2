"""Per-CTA timeline of k_gemv_mma (EZQ_GEMV_DBG=3): start, per-stage data-ready
and release times, end. Development aid."""
import ctypes as C
import os
import sys

import numpy as np
import torch

os.environ["EZQ_GEMV_DBG"] = os.environ.get("TLDBG", "8")
sys.path.insert(0, ".")
from paper_2403_02775_b200 import native as N  # noqa: E402
from paper_2403_02775_b200.native import Config  # noqa: E402

rows, cols, B = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
W = torch.randn(rows, cols, device="cuda") * 0.02
b = N.quantize_batch([W], Config(sigma_n=1e4), "outliers-only", out_mem=N.MEM_DEVICE)
plan = N.GemvPlan(b, 0)
x = torch.randn(B, rows, device="cuda").to(torch.bfloat16)
for _ in range(5):
    y = plan(x)
torch.cuda.synchronize()
ctas = 148
buf = np.zeros(64 * ctas, np.uint64)
N.lib().ezq_gemv_debug_timeline(buf.ctypes.data_as(C.c_void_p), ctas)
t = buf.reshape(ctas, 64).astype(np.int64)
t0 = t[:, 0].min()
start = (t[:, 0] - t0) / 1e3
end = (t[:, 62] - t0) / 1e3
total = t[:, 63]
print(f"CTA start: min {start.min():.2f} max {start.max():.2f} us; end: min {end.min():.2f} med {np.median(end):.2f} max {end.max():.2f} us")
print("stages per CTA:", np.bincount(total))
for i in [0, 1, 2, 3, 100]:
    n = int(total[i])
    ready = [(t[i, 2 + 2 * k] - t0) / 1e3 for k in range(min(n, 30))]
    rel = [(t[i, 3 + 2 * k] - t0) / 1e3 for k in range(min(n, 30))]
    print(f"cta {i} sm {t[i,1]}: start {start[i]:.2f} ready " + " ".join(f"{r:.2f}/{q:.2f}" for r, q in zip(ready, rel)) + f" end {end[i]:.2f}")
sm = t[:, 1]
per_sm_end = {}
for i in range(ctas):
    per_sm_end.setdefault(sm[i], []).append(end[i])
print("SMs:", len(per_sm_end), "max CTAs per SM:", max(len(v) for v in per_sm_end.values()))
arr = (t[:, 40:52] - t0) / 1e3
print("stage arrival (first `stages` stages) for CTAs 0..3:")
for i in range(4):
    print("  ", " ".join(f"{v:.2f}" for v in arr[i] if v > 0 and v < 1e6))

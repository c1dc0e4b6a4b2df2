"""Per-kernel-family device time of one quantize_batch of a bench workload (A/B aid).

python tools/fam_times.py [--workload llama-7b] [--reps 3] [--bits 4] [--sigma 3.0]
Prints ms per call for the whole call and each kernel family (in-library CUDA-event hooks).
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import layer_shapes  # noqa: E402
from paper_2403_02775_b200 import native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="llama-7b")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--bits", type=int, default=4)
ap.add_argument("--sigma", type=float, default=3.0)
a = ap.parse_args()
shapes = layer_shapes(a.workload)
Ws = []
for i, s in enumerate(shapes):
    g = torch.Generator(device="cuda").manual_seed(1234 + i)
    Ws.append(torch.randn(s, generator=g, device="cuda") * 0.02)
cfg = N.Config(bits=a.bits, sigma_n=a.sigma)
N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()
fams = ("stats", "detect", "qsort", "qrange", "qrange_stream", "seqerr", "pack")
N.profile_enable(True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(a.reps):
    N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) * 1e3 / a.reps
prof = {f: N.profile_read(f) for f in fams}
N.profile_enable(False)
print(f"{a.workload} bits={a.bits} sigma={a.sigma}: {ms:.2f} ms/call wall; " +
      " ".join(f"{f}={prof[f]['ms'] / a.reps:.2f}" for f in fams if prof[f]["launches"]))

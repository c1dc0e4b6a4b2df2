"""Counts K3s-vs-reference scale differences (selection near-ties) over every
tensor of one OPT-175B layer (test_property_bench_workload's generator)."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from oracle import pyoracle as O
from paper_2403_02775_b200 import native as N
from paper_2403_02775_b200.native import Config

shapes = [(12288, 12288)] * 4 + [(12288, 49152), (49152, 12288)]
g = torch.Generator(device="cuda").manual_seed(7)
Ws = [torch.randn(s, device="cuda", generator=g) * 0.02 for s in shapes]
qs = N.quantize_batch(Ws, Config())
tot_cols = tot_bad = 0
for i, (W, q) in enumerate(zip(Ws, qs)):
    t = time.time()
    r = O.quantize(W.cpu().numpy(), Config())
    a, b = q.scales.astype(np.float64), np.asarray(r["scales"], np.float64)
    bad = np.nonzero(a != b)[0]
    codes = int(np.count_nonzero(q.packed != np.asarray(r["packed"])))
    tot_cols += a.size
    tot_bad += bad.size
    print(i, shapes[i], "cols", a.size, "differ", bad.size,
          "maxrel %.3g" % (float(np.max(np.abs(a - b)[bad] / b[bad])) if bad.size else 0.0),
          "packed bytes differ", codes, "final_err equal", q.final_error == r["final_error"],
          "%.0fs" % (time.time() - t), flush=True)
print("total", tot_bad, "of", tot_cols, "columns")

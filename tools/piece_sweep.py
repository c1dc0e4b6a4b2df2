"""Scale mismatches vs the oracle across K3s row-piece counts (narrow tensors)."""
import sys, numpy as np
sys.path.insert(0, ".")
from oracle import pyoracle as O
from paper_2403_02775_b200 import native as N
from paper_2403_02775_b200.native import Config

cols = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for rows in [8192, 12288, 16384, 24576, 32768, 40960, 49152, 65536]:
    W = O.gaussian(rows, cols, 1000 + rows % 997, 0.02)
    q = N.quantize_tensor(W, Config())
    r = O.quantize(W, Config())
    a, b = q.scales.astype(np.float64), np.asarray(r["scales"], np.float64)
    bad = np.nonzero(a != b)[0]
    rel = float(np.max(np.abs(a - b) / b)) if len(bad) else 0.0
    print(rows, "bad", len(bad), "maxrel %.3g" % rel, "err", q.final_error == r["final_error"], q.final_error - r["final_error"],
          "cols", bad[:6].tolist(), flush=True)

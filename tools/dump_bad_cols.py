"""Finds the columns of the OPT-175B-layer 49152x12288 tensor (test_property_bench_workload's
generator) whose scale differs from the oracle; dumps their normals for offline analysis."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from oracle import pyoracle as O
from paper_2403_02775_b200 import native as N
from paper_2403_02775_b200.native import Config

shapes = [(12288, 12288)] * 4 + [(12288, 49152), (49152, 12288)]
g = torch.Generator(device="cuda").manual_seed(7)
Ws = [torch.randn(s, device="cuda", generator=g) * 0.02 for s in shapes]
Wd = Ws[5]
W = Wd.cpu().numpy()
del Ws
q = N.quantize_batch([Wd], Config())[0]
r = O.quantize(W, Config())
a, b = q.scales.astype(np.float64), np.asarray(r["scales"], np.float64)
bad = np.nonzero(a != b)[0]
print("bad", len(bad), bad[:20].tolist())
print("rel", (np.abs(a - b) / b)[bad][:20].tolist())
print("err", q.final_error, r["final_error"], q.rtn_error, r["rtn_error"])
o = q.outliers
mask = np.ones(W.shape, bool)
mask[o["row"], o["col"]] = False
out = {}
for c in bad[:8]:
    out[f"x{c}"] = W[mask[:, c], c]
    out[f"s{c}"] = np.array([a[c], b[c]])
np.savez("gpurun_out/bad_cols.npz", bad=bad, **out)

import sys; sys.path.insert(0,'.')
import numpy as np, torch
from oracle import pyoracle as O
from paper_2403_02775_b200 import native as N
from paper_2403_02775_b200.native import Config
for (rows, cols, sig) in [(64,40,100.0),(64,40,3.0),(512,40,100.0),(64,64,100.0)]:
    W = O.gaussian(rows, cols, 3, 0.02)
    b = N.quantize_batch([torch.from_numpy(W).cuda()], Config(steps=5, sigma_n=sig), out_mem=N.MEM_DEVICE)
    q = b.to_host(0); What = N.dequantize(q)
    plan = N.GemvPlan(b, 0)
    bad = []
    for i in range(rows):
        x = torch.zeros(1, rows, device='cuda'); x[0, i] = 1.0
        y = plan(x).cpu().numpy()[0]
        d = np.abs(y - What[i])
        if d.max() > 1e-6: bad.append((i, int(d.argmax()), float(d.max()), float(y[d.argmax()]), float(What[i][d.argmax()])))
    print(rows, cols, sig, "nout", len(q.outliers), "bad rows:", bad[:4], len(bad))

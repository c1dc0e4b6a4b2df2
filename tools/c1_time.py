"""Times the C1 pipeline repeatedly (device-resident input) for profiling."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
from oracle import refimpl as R
from paper_2403_02775_b200 import native as N
W = R.gaussian(4096, 4096, 1234)
R.plant_outliers(W, int(round(0.005 * W.size)), 10.0, 50.0, 5678)
Wd = torch.from_numpy(W).cuda()
cfg = N.Config()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for i in range(reps):
    torch.cuda.synchronize()
    t = time.time()
    b = N.quantize_batch([Wd], cfg, out_mem=N.MEM_DEVICE)
    torch.cuda.synchronize()
    print(f"rep {i}: {1e3*(time.time()-t):.2f} ms")
    b.close()

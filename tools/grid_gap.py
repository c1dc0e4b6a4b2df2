"""EasyQuant vs the brute-force grid optimum over a whole weight set
(the grid oracle at scale). For every column the
reference's grid (2000 scales in [s0/8, 1.25 s0] plus s0) is scanned on the
device (ezq_grid_oracle_batch, K3s tables); the tensor totals of EasyQuant's
final error and of the RTN error are compared with the sum of the per-column
grid optima. Prints one JSON line.

  python tools/grid_gap.py [--workload opt-1.3b] [--points 2000]
"""
import argparse
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import layer_shapes  # noqa: E402
from paper_2403_02775_b200 import native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="opt-1.3b")
    ap.add_argument("--points", type=int, default=2000)
    ap.add_argument("--sigma", type=float, default=3.0)
    a = ap.parse_args()
    shapes = layer_shapes(a.workload)
    g = torch.Generator(device="cuda").manual_seed(1)
    Ws = [torch.randn(s, generator=g, device="cuda") * 0.02 for s in shapes]
    cfg = N.Config(sigma_n=a.sigma)
    b = N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE)
    rtn = sum(b[i].rtn_error for i in range(len(b)))
    fin = sum(b[i].final_error for i in range(len(b)))
    b.close()
    N.grid_oracle_batch(Ws[:6], cfg, a.points)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = N.grid_oracle_batch(Ws, cfg, a.points)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    opt = float(sum(e.sum() for _, e in res))
    cols = sum(s[1] for s in shapes)
    print(json.dumps({
        "workload": a.workload, "columns": cols, "grid_points": a.points + 1, "sigma_n": a.sigma,
        "grid_oracle_s": dt, "scales_per_s": cols * (a.points + 1) / dt,
        "rtn_error": rtn, "easyquant_error": fin, "grid_optimum_error": opt,
        "easyquant_over_optimum": fin / opt, "rtn_over_optimum": rtn / opt,
    }))


if __name__ == "__main__":
    main()

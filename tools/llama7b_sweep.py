"""configs[2]: LLaMA-7B-shaped weight set (32 layers x 4 x 4096^2 + 3 x
4096x11008), 4-bit and 3-bit, outlier-threshold sweep 0.1-1% (sigma_n from
the two-sided Gaussian tail: 3.2905 -> 0.1%, 2.8070 -> 0.5%, 2.5758 -> 1%).
The weights stay resident in HBM across the sweep (the batched sweep of
SURVEY §8f #2); each point is one quantize_batch of the whole set, timed with
CUDA events. Prints one JSON line per point.

  python tools/llama7b_sweep.py [--layers 32]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_02775_b200 import native as N  # noqa: E402
from paper_2403_02775_b200.native import Config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    a = ap.parse_args()
    N.set_device(0)
    h, ffn = 4096, 11008
    shapes = ([(h, h)] * 4 + [(h, ffn), (h, ffn), (ffn, h)]) * a.layers
    g = torch.Generator(device="cuda").manual_seed(7)
    Ws = [torch.randn(s, generator=g, device="cuda") * 0.02 for s in shapes]
    weights = sum(r * c for r, c in shapes)
    torch.cuda.synchronize()
    for bits in (4, 3):
        for sigma in (3.2905, 2.8070, 2.5758):
            cfg = Config(bits=bits, sigma_n=sigma)
            N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()  # warm (allocations, caches)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b = N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            n_out = sum(b[i].n_outliers for i in range(len(b)))
            rtn = sum(b[i].rtn_error for i in range(len(b)))
            fin = sum(b[i].final_error for i in range(len(b)))
            b.close()
            print(json.dumps({"workload": f"LLaMA-7B-shaped, {a.layers} layers", "bits": bits,
                              "sigma_n": sigma, "weights": weights,
                              "outlier_fraction": n_out / weights, "ms": ms,
                              "weights_per_s": weights / (ms / 1e3),
                              "error_reduction_pct": 100.0 * (rtn - fin) / rtn}), flush=True)


if __name__ == "__main__":
    main()

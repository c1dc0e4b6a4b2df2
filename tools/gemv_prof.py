"""Single-configuration GEMV timing (development aid, ncu-friendly).

python tools/gemv_prof.py --rows 4096 --cols 11008 --batch 1 --ratio 0.01
Prints us/GEMV (CUDA-graph replay over `copies` rotated weight copies, CUDA
events) and the effective HBM GB/s of the algorithmic bytes.
"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2403_02775_b200 import native as N  # noqa: E402
from paper_2403_02775_b200.native import Config  # noqa: E402

SIG = {0.0: 1.0e4, 0.005: 2.8070, 0.01: 2.5758}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--cols", type=int, default=11008)
    ap.add_argument("--batch", type=int, nargs="+", default=[1])
    ap.add_argument("--ratio", type=float, nargs="+", default=[0.0])
    ap.add_argument("--copies", type=int, default=8)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--dtype", default="bfloat16")
    ap.add_argument("--plain", action="store_true", help="no graph: launch a few times (for ncu)")
    ap.add_argument("--odt", default="float32", help="outlier value dtype (float32 / float16)")
    a = ap.parse_args()
    gen = torch.Generator(device="cuda").manual_seed(99)
    r, c = a.rows, a.cols
    dense = [(torch.randn(r, c, generator=gen, device="cuda") * 0.02) for _ in range(a.copies)]
    for ratio in a.ratio:
        b = N.quantize_batch(dense, Config(sigma_n=SIG[ratio]), "outliers-only", out_mem=N.MEM_DEVICE)
        plans = [N.GemvPlan(b, i, outlier_dtype=a.odt) for i in range(a.copies)]
        n_out = sum(b[i].n_outliers for i in range(a.copies)) / a.copies
        for B in a.batch:
            x = torch.randn(B, r, generator=gen, device="cuda").to(getattr(torch, a.dtype))
            y = torch.empty(B, c, device="cuda", dtype=torch.float32)
            if a.plain:
                for _ in range(3):
                    for p in plans:
                        p(x, y)
                torch.cuda.synchronize()
                continue
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                for p in plans:
                    p(x, y)
            torch.cuda.current_stream().wait_stream(s)
            with torch.cuda.graph(g):
                for p in plans:
                    p(x, y)
            for _ in range(3):
                g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / a.reps / a.copies * 1e3
            vb = 6 if a.odt == "float32" else 4  # value + u16 row
            nbytes = r * c / 2 + 4 * c + vb * n_out + x.element_size() * B * r + 4 * B * c
            print(f"{r}x{c} B={B} ratio={ratio} n_out={n_out:.0f}: {us:.2f} us  {nbytes / us / 1e3:.0f} GB/s")
        for p in plans:
            p.close()
        b.close()


if __name__ == "__main__":
    main()

"""A/B timing of the q_range kernels on C1-like and OPT-like tensors (dev aid)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2403_02775_b200 import native as N
shapes = [(2048, 2048)] * 8 + [(8192, 2048)] * 2 + [(4096, 4096)] * 2
g = torch.Generator(device="cuda").manual_seed(3)
for rows, cols in sorted(set(shapes)):
    Ws = [torch.randn(rows, cols, generator=g, device="cuda") * 0.02 for _ in range(4)]
    for steps in (0, 200):
        cfg = N.Config(steps=steps)
        N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()
        N.profile_enable(True)
        torch.cuda.synchronize(); t = time.perf_counter()
        N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        prof = {"ms": N.profile_read("qrange")["ms"] + N.profile_read("qsort")["ms"]}
        N.profile_enable(False)
        print(f"{rows}x{cols} x4 steps={steps}: total {dt*1e3:.1f} ms, qrange {prof['ms']:.1f} ms")

"""PCIe ceiling for the end-to-end path (dev aid): pinned host -> device copy
bandwidth of the LLaMA-7B weight set (25.9 GB) in 384 MB chunks on one
stream, against one ezq_quantize_batch call with host inputs and outputs.
python tools/h2d_ceiling.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import layer_shapes  # noqa: E402
from paper_2403_02775_b200 import native as N  # noqa: E402

shapes = layer_shapes("llama-7b")
g = torch.Generator(device="cuda").manual_seed(1)
hosts = []
for s in shapes:
    h = torch.empty(s, dtype=torch.float32, pin_memory=True)
    h.copy_(torch.randn(s, generator=g, device="cuda") * 0.02)
    hosts.append(h)
tot = sum(h.numel() * 4 for h in hosts)
dev = torch.empty(384 << 20 >> 2, dtype=torch.float32, device="cuda")
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for h in hosts:
        f = h.view(-1)
        for o in range(0, f.numel(), dev.numel()):
            n = min(dev.numel(), f.numel() - o)
            dev[:n].copy_(f[o:o + n], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"H2D {tot / 1e9:.1f} GB in {dt * 1e3:.0f} ms: {tot / dt / 1e9:.1f} GB/s")
Wn = [h.numpy() for h in hosts]
cfg = N.Config()
for rep in range(3):
    t0 = time.perf_counter()
    q = N.quantize_batch(Wn, cfg)
    del q
    dt = time.perf_counter() - t0
    print(f"quantize_batch host->host: {dt * 1e3:.0f} ms ({tot / dt / 1e9:.1f} GB/s of inputs)")

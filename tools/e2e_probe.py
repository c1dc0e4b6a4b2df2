"""Where does the e2e time go? OPT-1.3B set: device in/device out, device in/host
out, host in/host out (development aid)."""
import sys, time
import torch
sys.path.insert(0, ".")
from bench import layer_shapes
from paper_2403_02775_b200 import native as N
shapes = layer_shapes("opt-1.3b")
g = torch.Generator(device="cuda").manual_seed(1)
Ws = [torch.randn(s, generator=g, device="cuda") * 0.02 for s in shapes]
Wn = [w.cpu().pin_memory().numpy() for w in Ws]
cfg = N.Config()
def t(fn, k=2):
    fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
print("dev->dev  %.1f ms" % t(lambda: N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()))
print("dev->host %.1f ms" % t(lambda: N.quantize_batch(Ws, cfg)))
print("host->dev %.1f ms" % t(lambda: N.quantize_batch(Wn, cfg, out_mem=N.MEM_DEVICE).close()))
print("host->host %.1f ms" % t(lambda: N.quantize_batch(Wn, cfg)))

import sys, torch
sys.path.insert(0, ".")
from paper_2403_02775_b200 import native as N
shapes = [((8192, 2048), 24), ((2048, 2048), 96), ((2048, 8192), 24), ((8192, 2048), 24)]
if len(sys.argv) > 1:
    shapes = shapes[:int(sys.argv[1])]
for shape, cnt in shapes:
    g = torch.Generator(device="cuda").manual_seed(1)
    Ws = [torch.randn(shape, generator=g, device="cuda") * 0.02 for _ in range(cnt)]
    torch.cuda.synchronize()
    try:
        N.quantize_batch(Ws, N.Config(), out_mem=N.MEM_DEVICE).close()
        torch.cuda.synchronize()
        print(shape, cnt, "ok", flush=True)
    except Exception as e:
        print(shape, cnt, "FAIL", e, flush=True)
        break

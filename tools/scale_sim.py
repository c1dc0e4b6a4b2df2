"""Strong-scaling estimate on ONE GPU (this environment has one): the bench's LPT partition of
the LLaMA-7B set (driver.lpt_partition) is quantized rank by rank, and the N-GPU step time is
the slowest rank's share (there is no collective on the data path, so a rank's time does not
depend on the others). This measures the partition's balance and the per-call fixed costs at
1/N of the work; it is not a multi-GPU run (NVLink/host contention is not modelled).

  python tools/scale_sim.py [--workload llama-7b] [--ranks 1 2 4 8]
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from bench import layer_shapes  # noqa: E402
from paper_2403_02775_b200 import native as N  # noqa: E402
from paper_2403_02775_b200.driver import lpt_partition  # noqa: E402
from paper_2403_02775_b200.native import Config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="llama-7b")
ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
shapes = layer_shapes(a.workload)
total = sum(r * c for r, c in shapes)
cfg = Config()


def gen(i):
    g = torch.Generator(device="cuda").manual_seed(1234 + i)
    return torch.randn(shapes[i], generator=g, device="cuda") * 0.02


rows = []
for n in a.ranks:
    times = []
    for rank, mine in enumerate(lpt_partition([r * c for r, c in shapes], n)):
        Ws = [gen(i) for i in mine]
        N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()  # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / a.reps)
        del Ws
    step = max(times)
    rows.append({"ranks": n, "rank_ms": times, "step_ms": step, "weights_per_s": total / (step * 1e-3)})
base = rows[0]["weights_per_s"] if rows and rows[0]["ranks"] == 1 else None
for r in rows:
    r["efficiency_vs_1"] = r["weights_per_s"] / (base * r["ranks"]) if base else None
    print(json.dumps(r), flush=True)

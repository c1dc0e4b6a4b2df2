"""configs[3]: quantize a full OPT-175B-shaped weight set (96 layers, hidden
12288: 4 x 12288^2 + 12288x49152 + 49152x12288 per layer, 174B weights) with
~1% outliers (sigma_n = 2.5758, the two-sided 1% point of a Gaussian), the
layers sharded round-robin over the ranks of a torchrun job (one process per
GPU, no collective on the data path). Weights are synthetic and generated
on the device one layer at a time (the model does not fit in HBM), so the
timing is the quantizer itself: device time per layer (CUDA events) summed,
plus the wall clock of the whole run. Rank 0 prints one JSON line.

  python tools/opt175b_run.py [--layers 96]
  python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 tools/opt175b_run.py
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_02775_b200 import native as N  # noqa: E402
from paper_2403_02775_b200.native import Config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=96)
    ap.add_argument("--sigma", type=float, default=2.5758)
    a = ap.parse_args()
    rank, local, world = (int(os.environ.get(k, d)) for k, d in
                          (("RANK", 0), ("LOCAL_RANK", 0), ("WORLD_SIZE", 1)))
    torch.cuda.set_device(local)
    N.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    h, ffn = 12288, 49152
    shapes = [(h, h)] * 4 + [(h, ffn), (ffn, h)]
    cfg = Config(sigma_n=a.sigma)
    mine = list(range(rank, a.layers, world))
    dev_ms, weights, outliers, worst = 0.0, 0, 0, 0.0
    t0 = time.perf_counter()
    for layer in mine:
        g = torch.Generator(device="cuda").manual_seed(1000 + layer)
        Ws = [torch.randn(s, generator=g, device="cuda") * 0.02 for s in shapes]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b = N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE)
        e1.record()
        torch.cuda.synchronize()
        dev_ms += e0.elapsed_time(e1)
        for i, s in enumerate(shapes):
            q = b[i]
            weights += s[0] * s[1]
            outliers += q.n_outliers
            assert q.final_error <= q.rtn_error
            worst = max(worst, q.final_error / q.rtn_error if q.rtn_error else 0.0)
        b.close()
        del Ws
    wall = time.perf_counter() - t0
    tot = torch.tensor([dev_ms, wall, float(weights), float(outliers)], dtype=torch.float64, device="cuda")
    if world > 1:
        import torch.distributed as dist
        mx = tot.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = tot.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        dev_ms, wall = mx[0].item(), mx[1].item()
        weights, outliers = int(sm[2].item()), int(sm[3].item())
    if rank == 0:
        print(json.dumps({
            "workload": f"OPT-175B-shaped, {a.layers} layers x 6 matrices, 4-bit, sigma_n {a.sigma}",
            "n_gpus": world, "weights": weights, "outlier_fraction": outliers / weights,
            "device_s_max_rank": dev_ms / 1e3, "wall_s_max_rank": wall,
            "weights_per_s_device": weights / (dev_ms / 1e3),
            "worst_final_over_rtn": worst,
            "paper_claim": "< 10 min on 8 GPUs (EasyQuant, arXiv 2403.02775)",
        }))


if __name__ == "__main__":
    main()

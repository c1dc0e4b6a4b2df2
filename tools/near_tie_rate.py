"""Selection near-ties over every tensor of one OPT-175B layer (test_property_bench_workload's
generator), against the oracle (C restatement of the reference): columns whose scale differs
(must be 0), columns the K3s loop flagged and resolved in reference order, whole-loop
fallbacks, and what the certification costs (the same batch with EZQ_TIE_CAP=0, i.e. no
near-tie tracking, timed in a subprocess). One JSON line per sigma_n.

  python tools/near_tie_rate.py [sigma_n ...]          (default: 3.0 2.5758)
"""
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import pyoracle as O  # noqa: E402
from paper_2403_02775_b200 import native as N  # noqa: E402
from paper_2403_02775_b200.native import Config  # noqa: E402

shapes = [(12288, 12288)] * 4 + [(12288, 49152), (49152, 12288)]


def layer():
    g = torch.Generator(device="cuda").manual_seed(7)
    return [torch.randn(s, device="cuda", generator=g) * 0.02 for s in shapes]


def device_ms(Ws, cfg, reps=2):
    N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        N.quantize_batch(Ws, cfg, out_mem=N.MEM_DEVICE).close()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "--time-only":
    print(device_ms(layer(), Config(sigma_n=float(sys.argv[2]))))
    sys.exit(0)

for sig in [float(a) for a in sys.argv[1:]] or [3.0, 2.5758]:
    Ws = layer()
    cfg = Config(sigma_n=sig)
    t0 = N.tie_stats()
    qs = N.quantize_batch(Ws, cfg)
    t1 = N.tie_stats()
    ms_on = device_ms(Ws, cfg)
    env = dict(os.environ, EZQ_TIE_CAP="0")
    ms_off = float(subprocess.run([sys.executable, __file__, "--time-only", str(sig)], env=env, capture_output=True,
                                  text=True, check=True).stdout.split()[-1])
    tot_cols = tot_bad = codes = 0
    for W, q in zip(Ws, qs):
        r = O.quantize(W.cpu().numpy(), cfg)
        a, b = q.scales.view(np.uint32), np.asarray(r["scales"]).view(np.uint32)
        tot_cols += a.size
        tot_bad += int(np.count_nonzero(a != b))
        codes += int(np.count_nonzero(q.packed != np.asarray(r["packed"])))
        assert q.final_error == r["final_error"] and q.rtn_error == r["rtn_error"]
    print(json.dumps({"workload": "one OPT-175B layer (4 x 12288^2, 12288x49152, 49152x12288)", "sigma_n": sig,
                      "columns": tot_cols, "scale_mismatches_vs_oracle": tot_bad, "packed_bytes_differ": codes,
                      "near_tie_columns_resolved": t1[0] - t0[0], "whole_loop_fallbacks": t1[1] - t0[1],
                      "device_ms_with_certification": ms_on, "device_ms_without": ms_off,
                      "certification_cost_ms": ms_on - ms_off}), flush=True)
    del Ws, qs
    torch.cuda.empty_cache()

"""Dense 3-bit codec throughput (§8f #4): pack / unpack / dequantize from the
dense stream vs dequantize from the byte-per-level codes, on a device-resident
3-bit artifact (CUDA events around `reps` calls; algorithmic bytes per call).

python tools/dense3_bench.py [--rows 11008 --cols 4096 --reps 50]
"""
import argparse
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_02775_b200 import native as N  # noqa: E402
from paper_2403_02775_b200.native import Config, check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=11008)
ap.add_argument("--cols", type=int, default=4096)
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
rows, cols = a.rows, a.cols
n = rows * cols
g = torch.Generator(device="cuda").manual_seed(3)
Wd = torch.randn(rows, cols, generator=g, device="cuda") * 0.02
b = N.quantize_batch([Wd], Config(bits=3, sigma_n=2.5758, steps=20), out_mem=N.MEM_DEVICE)
codes = torch.from_numpy(b.to_host(0).packed.copy()).cuda()
dense = N.pack_dense3(codes)
back = torch.empty_like(codes)
out = torch.empty(rows, cols, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / a.reps  # us per call (includes the host sync of each call)


d3 = N.dense3_size(n)
res = {"shape": f"{rows}x{cols}", "weights": n, "dense3_bytes": d3, "byte_codes_bytes": n,
       "n_outliers": int(b[0].n_outliers)}
res["pack_us"] = timed(lambda: check(lib().ezq_pack_dense3(codes.data_ptr(), n, dense.data_ptr(), N.MEM_DEVICE, st)))
res["unpack_us"] = timed(lambda: check(lib().ezq_unpack_dense3(dense.data_ptr(), n, back.data_ptr(), N.MEM_DEVICE, st)))
res["dequant_dense3_us"] = timed(lambda: b.dequantize_dense3_into(0, dense, out))
res["dequant_bytes_us"] = timed(lambda: b.dequantize_into(0, out))
# device-side kernel time via the in-library profile (family "dense3" / "dequant")
N.profile_enable(True)
for _ in range(a.reps):
    b.dequantize_dense3_into(0, dense, out)
    b.dequantize_into(0, out)
pr, pb = N.profile_read("dense3"), N.profile_read("dequant")
N.profile_enable(False)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6538.6
for key, prof, codes_b in (("dense3", pr, d3), ("bytes", pb, n)):
    us = prof["ms"] * 1e3 / a.reps
    alg = codes_b + 4 * cols + 4 * n + 12 * res["n_outliers"]  # codes + scales + floats out + COO entries
    res[f"dequant_{key}_device_us"] = us
    res[f"dequant_{key}_device_gbs"] = alg / (us * 1e-6) / 1e9
    res[f"dequant_{key}_hbm_frac"] = res[f"dequant_{key}_device_gbs"] / peak
print(json.dumps(res))
b.close()

"""Ad-hoc GPU-vs-reference parity sweep (development aid; the formal gate is
tests/test_gpu_parity.py). Prints per-case mismatch statistics."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import refimpl as R  # noqa: E402
from paper_2403_02775_b200 import native as N  # noqa: E402


def cmp_case(name, W, cfg, mode="easyquant"):
    t0 = time.time()
    q = N.quantize_tensor(W, cfg, mode)
    tg = time.time() - t0
    t0 = time.time()
    r = R.quantize(W, cfg, mode)
    tr = time.time() - t0
    same_out = np.array_equal(q.outliers, r.outliers)
    sdiff = np.nonzero(q.scales != r.scales)[0]
    rel = np.max(np.abs(q.scales.astype(np.float64) - r.scales) / r.scales) if len(sdiff) else 0.0
    pk_eq = np.array_equal(q.packed, r.packed)
    nib_diff = 0
    if not pk_eq:
        a, b = q.packed, r.packed
        if cfg.bits == 4:
            nib_diff = int(np.sum((a & 15) != (b & 15)) + np.sum((a >> 4) != (b >> 4)))
        else:
            nib_diff = int(np.sum(a != b))
    print(f"{name:34s} mode={mode:13s} gpu {tg*1e3:8.1f} ms ref {tr*1e3:8.1f} ms | outl {len(q.outliers)} eq={same_out} "
          f"mean_eq={q.mean == r.mean} std_eq={q.stddev == r.stddev} | scales diff {len(sdiff)}/{W.shape[1]} maxrel {rel:.2e} | "
          f"codes diff {nib_diff} | rtn {q.rtn_error == r.rtn_error} fin {q.final_error == r.final_error} "
          f"({q.final_error:.6g} vs {r.final_error:.6g})")
    d = N.dequantize(q)
    dr = r.dequantize(*W.shape)
    print(f"{'':34s} dequant eq={np.array_equal(d.view(np.uint32), dr.view(np.uint32))}")
    return len(sdiff) == 0 and pk_eq and same_out


def main():
    print("devices", N.device_count())
    cfg = N.Config()
    ok = True
    W = R.gaussian(64, 64, 31)
    ok &= cmp_case("64x64", W, cfg)
    for mode in ("rtn", "outliers-only"):
        ok &= cmp_case("64x64", W, cfg, mode)
    W = R.gaussian(96, 64, 71, 0.05)
    R.plant_outliers(W, 31, 0.5, 2.5, 72)
    c2 = N.Config(steps=60)
    ok &= cmp_case("96x64 planted steps60", W, c2)
    W = R.gaussian(513, 77, 5, 0.02)
    ok &= cmp_case("513x77 sigma.02", W, cfg)
    ok &= cmp_case("513x77 k3", W, N.Config(bits=3))
    ok &= cmp_case("513x77 fixed", W, N.Config(select="fixed"))
    W = R.gaussian(2048, 256, 7)
    ok &= cmp_case("2048x256", W, cfg)
    W = R.gaussian(8192, 64, 9, 0.02)
    ok &= cmp_case("8192x64 lr1e-4", W, N.Config(lr=1e-4))
    W = R.gaussian(12288, 32, 19, 0.02)
    ok &= cmp_case("12288x32", W, cfg)
    W = R.gaussian(4096, 4096, 1234)
    R.plant_outliers(W, int(round(0.005 * W.size)), 10.0, 50.0, 5678)
    ok &= cmp_case("C1 4096x4096 planted", W, cfg)
    # channel API
    x = R.gaussian(1, 1024, 7)[0]
    a = N.optimize_channel(x, None, N.Config(lr=3e-3), True)
    b = R.optimize_channel(x, None, N.Config(lr=3e-3), True)
    print("optimize_channel exact:", a["scale"] == b["scale"], np.array_equal(a["trace_scale"], b["trace_scale"]),
          np.array_equal(a["trace_error"], b["trace_error"]))
    print("brute force exact:", N.brute_force_scale(x, None, cfg, 2000) == R.brute_force_scale(x, None, cfg, 2000))
    print("ALL OK" if ok else "MISMATCH")


if __name__ == "__main__":
    main()

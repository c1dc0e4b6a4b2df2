"""Generates tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libezq_ref.so, compiled from /root/reference/proj by
oracle/Makefile). Run here (where /root/reference exists):

    make -C oracle ref && python tools/make_golden.py

The fixtures hold inputs AND reference outputs, so the GPU box (which has no
/root/reference) can pin both the C restatement and the CUDA path.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import refimpl as R  # noqa: E402
from paper_2403_02775_b200.native import Config  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")


def cfg_arr(c: Config):
    return np.array([c.bits, c.sigma_n, c.lr, c.beta1, c.beta2, c.eps, c.steps,
                     1 if c.select == "fixed" else 0, c.select_step], np.float64)


def quant_case(name, W, cfg, mode):
    q = R.quantize(W, cfg, mode)
    deq = q.dequantize(*W.shape)
    np.savez_compressed(os.path.join(OUT, f"quant_{name}.npz"), W=W, cfg=cfg_arr(cfg),
                        mode=np.array(mode), packed=q.packed, scales=q.scales,
                        outliers=q.outliers, mean=q.mean, stddev=q.stddev,
                        rtn_error=q.rtn_error, final_error=q.final_error, dequant=deq)


def main():
    os.makedirs(OUT, exist_ok=True)
    d = Config()
    # Matrices of the reference's unit tests (test_pipeline.cpp / test_stats.cpp).
    quant_case("kat_1x5", np.array([[0, 0, 0, 0, 100]], np.float32), Config(sigma_n=2.0), "easyquant")
    quant_case("const_16x12", np.full((16, 12), 2.0, np.float32), d, "easyquant")
    quant_case("grid_4x1_rtn", np.array([[0.5], [-1.5], [4.0], [2.0]], np.float32), d, "rtn")
    quant_case("alloutlier_2x2", np.array([[100, 1], [-100, 1]], np.float32), Config(sigma_n=1.0),
               "easyquant")
    quant_case("golden_1x2", np.array([[1.0, 100.0]], np.float32), Config(sigma_n=1.0), "easyquant")
    W = R.gaussian(64, 64, 31)
    for mode in ("easyquant", "rtn", "outliers-only"):
        quant_case(f"g64_{mode}", W, d, mode)
    W = R.gaussian(96, 64, 71, 0.05)
    R.plant_outliers(W, 31, 0.5, 2.5, 72)
    quant_case("planted96x64_s60", W, Config(steps=60), "easyquant")
    W = R.gaussian(513, 77, 5, 0.02)
    quant_case("s02_513x77_k3", W, Config(bits=3), "easyquant")
    quant_case("s02_513x77_fixed", W, Config(select="fixed"), "easyquant")
    quant_case("s02_513x77_k8", W, Config(bits=8), "easyquant")
    quant_case("s02_513x77_k2", W, Config(bits=2), "outliers-only")
    quant_case("row_1x37", R.gaussian(1, 37, 63), d, "easyquant")
    quant_case("col_53x1", R.gaussian(53, 1, 64), d, "easyquant")
    W = R.gaussian(48, 56, 41, 0.04)
    R.plant_outliers(W, 13, 0.4, 2.0, 1041)
    quant_case("planted48x56", W, d, "easyquant")
    # Stats KATs (test_stats.cpp:27-53) + ragged chunk sizes.
    stats = {}
    for name, M in [("kat", np.array([[0, 0, 0, 0, 100]], np.float32)),
                    ("pop", np.array([[1.0, 3.0]], np.float32)),
                    ("single", np.array([[-2.5]], np.float32)),
                    ("ragged", R.gaussian(123, 217, 1, 0.05)),
                    ("multi_chunk", R.gaussian(301, 157, 7))]:
        st = R.tensor_stats(M)
        stats[name + "_W"] = M
        stats[name + "_out"] = np.array([st["mean"], st["stddev"], st["max_abs"]])
    np.savez_compressed(os.path.join(OUT, "stats.npz"), **stats)
    # Channel traces (test_optimize.cpp / acceptance criterion 8).
    x = R.gaussian(1, 1024, 7)[0]
    tr = R.optimize_channel(x, None, Config(lr=3e-3), True)
    bf = R.brute_force_scale(x, None, Config(), 2000)
    ev = R.channel_eval(x, None, 0.11, Config())
    np.savez_compressed(os.path.join(OUT, "channel.npz"), x=x, trace_scale=tr["trace_scale"],
                        trace_error=tr["trace_error"], scale=tr["scale"],
                        initial_error=tr["initial_error"], final_error=tr["final_error"],
                        best_step=tr["best_step"], bf=np.array(bf), ev=np.array(ev))
    # The 89-byte .ezqt golden fixture of test_io.cpp:122-151.
    q = R.quantize(np.array([[1.0, 100.0]], np.float32), Config(sigma_n=1.0), "easyquant")
    b = q.encode()
    assert len(b) == 89, len(b)
    with open(os.path.join(OUT, "golden_1x2.ezqt"), "wb") as f:
        f.write(b)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()

"""CPU: the drop-in boundary. libezq_b200.so (C-ABI) and libezquant.so (C++
drop-in) load, export every entry point include/ezquant_c.h declares and every
reference API function include/ezquant/*.hpp declares; compute entry points
fail loudly (EZQ_ERR_NO_DEVICE) without a GPU -- there is no CPU fallback;
the host-only scalar utilities match the oracle / reference semantics."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, _cuda_available
from paper_2403_02775_b200.native import Config

HEADER = os.path.join(ROOT, "include", "ezquant_c.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ezq_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_api():
    syms = declared_symbols()
    for s in ("ezq_quantize_tensor", "ezq_quantize_batch", "ezq_dequantize_tensor",
              "ezq_tensor_stats", "ezq_detect_outliers", "ezq_optimize_channel", "ezq_gemv",
              "ezq_last_error", "ezq_free", "ezq_reconstruction_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(N):
    lib = C.CDLL(N.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_cpp_dropin_exports_reference_api(N):
    so = os.path.join(os.path.dirname(N.LIB_PATH), "libezquant.so")
    out = subprocess.run(["nm", "-DC", "--defined-only", so], capture_output=True, text=True,
                         check=True).stdout
    for fn in ("ezquant::quantize_tensor(", "ezquant::easyquant_tensor(", "ezquant::rtn_tensor(",
               "ezquant::dequantize_tensor(", "ezquant::serial::quantize_tensor(",
               "ezquant::serial::dequantize_tensor(", "ezquant::tensor_stats(",
               "ezquant::serial::tensor_stats(", "ezquant::detect_outliers(",
               "ezquant::outlier_rows_by_column(", "ezquant::normal_mask_apply(",
               "ezquant::scatter_outliers(", "ezquant::initial_scale(", "ezquant::quantize_channel(",
               "ezquant::dequantize_channel(", "ezquant::reconstruction_error(", "ezquant::pack_levels(",
               "ezquant::unpack_levels(", "ezquant::packed_size(", "ezquant::adam_step(",
               "ezquant::channel_error(", "ezquant::range_gradient(", "ezquant::channel_eval(",
               "ezquant::optimize_channel_range(", "ezquant::brute_force_optimal_scale(",
               "ezquant::parse_quant_mode(", "ezquant::quant_mode_name(",
               "ezquant::DenseMatrix::validate() const", "ezquant::QuantConfig::validate() const"):
        assert fn in out, fn


@pytest.mark.skipif(_cuda_available(), reason="checks the no-device path")
def test_no_cpu_fallback(N):
    W = np.ones((4, 4), np.float32)
    with pytest.raises(N.EzqError) as e:
        N.quantize_tensor(W, Config())
    assert e.value.code == N.NO_DEVICE
    with pytest.raises(N.EzqError):
        N.tensor_stats(W)
    with pytest.raises(N.EzqError):
        N.optimize_channel(np.ones(8, np.float32), None, Config())


def test_config_validation(N):  # types.cpp:23-40 messages
    N.config_validate(Config())
    for bad, msg in [(Config(bits=9), "bits must be in [2, 8], got 9"),
                     (Config(sigma_n=-1.0), "sigma_n must be finite and >= 0"),
                     (Config(lr=0.0), "lr must be finite and > 0"),
                     (Config(beta1=1.0), "adam_beta1 must be in [0, 1)"),
                     (Config(beta2=-0.1), "adam_beta2 must be in [0, 1)"),
                     (Config(eps=0.0), "adam_eps must be > 0"),
                     (Config(steps=-1), "steps must be >= 0"),
                     (Config(select_step=-2), "select_step must be >= 0")]:
        with pytest.raises(N.InvalidArgument) as e:
            N.config_validate(bad)
        assert e.value.msg == msg


def test_host_utilities_match_oracle(N, O):
    rng = np.random.default_rng(3)
    for bits in (2, 3, 4, 5, 8):
        lmin, lmax = 1 - (1 << (bits - 1)), 1 << (bits - 1)
        lv = rng.integers(lmin, lmax + 1, 999).astype(np.int16)
        pk = N.pack_levels(lv, bits)
        assert np.array_equal(pk, O.pack_levels(lv, bits))
        assert np.array_equal(N.unpack_levels(pk, 999, bits), lv)
        assert N.packed_size(999, bits) == (500 if bits == 4 else 999)
    assert N.pack_levels([-7, 8], 4).tolist() == [0xF0]
    with pytest.raises(N.InvalidArgument):
        N.pack_levels([-8], 4)
    with pytest.raises(N.InvalidArgument):
        N.unpack_levels(np.array([0, 1], np.uint8), 5, 4)
    x = rng.standard_normal(300).astype(np.float32)
    assert N.initial_scale(x, Config()) == O.initial_scale(x, 4)
    for g in (0.0, 1.0, -3.5e-2, 7e3):
        a, b = {"m": 0.1, "v": 0.2, "t": 3}, {"m": 0.1, "v": 0.2, "t": 3}
        assert N.adam_step(a, 0.37, g, Config()) == O.adam_step(b, 0.37, g, Config())
        assert a == b
    lv = rng.integers(-7, 9, 50).astype(np.int16)
    d = N.dequantize_channel(lv, 0.1234)
    assert np.array_equal(d, (0.1234 * lv.astype(np.float64)).astype(np.float32))

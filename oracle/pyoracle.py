"""TEST INFRASTRUCTURE ONLY: ctypes binding of the C restatement
(oracle/ezq_oracle.c -> oracle/build/libezq_oracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module, and only as the checker or the
timed CPU baseline. The library is (re)built with gcc on first use when
missing, so it works on a GPU box without /root/reference.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "build", "libezq_oracle.so")
OUTLIER_DTYPE = np.dtype([("row", "<u4"), ("col", "<u4"), ("value", "<f4")])
MODES = {"easyquant": 0, "rtn": 1, "outliers-only": 2}


class OConfig(C.Structure):  # same layout as ezq_config (include/ezquant_c.h)
    _fields_ = [("bits", C.c_int32), ("sigma_n", C.c_float), ("lr", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("steps", C.c_int32), ("select", C.c_int32), ("select_step", C.c_int32),
                ("reserved", C.c_int32), ("seed", C.c_uint64)]


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "ezq_oracle.c")
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    return SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(SO)
        P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int, C.c_double
        L.ezqo_gaussian.argtypes = [P, I64, C.c_uint64, D]
        L.ezqo_plant_outliers.argtypes = [P, I64, I64, D, D, C.c_uint64]
        L.ezqo_tensor_stats.argtypes = [P, I64, C.POINTER(D), C.POINTER(D), C.POINTER(D)]
        L.ezqo_detect_outliers.argtypes = [P, I64, I64, C.c_float, P, C.POINTER(D), C.POINTER(D)]
        L.ezqo_detect_outliers.restype = I64
        L.ezqo_initial_scale.argtypes = [P, I64, I32]
        L.ezqo_initial_scale.restype = D
        L.ezqo_level_of.argtypes = [D, D, I32, I32]
        L.ezqo_eval_dense.argtypes = [P, I64, D, I32, I32, C.POINTER(D), C.POINTER(D)]
        L.ezqo_adam_step.argtypes = [C.POINTER(D), C.POINTER(D), C.POINTER(I64), D, D,
                                     C.POINTER(OConfig)]
        L.ezqo_adam_step.restype = D
        L.ezqo_optimize_channel.argtypes = [P, I64, C.POINTER(OConfig), C.POINTER(D), C.POINTER(D),
                                            C.POINTER(C.c_int), P, P]
        L.ezqo_optimize_channel.restype = C.c_float
        L.ezqo_brute_force.argtypes = [P, I64, C.POINTER(OConfig), I32, C.POINTER(D), C.POINTER(D)]
        L.ezqo_quantize.argtypes = [P, I64, I64, C.POINTER(OConfig), I32, I32, P, P, P, I64,
                                    C.POINTER(D), C.POINTER(D), C.POINTER(D), C.POINTER(D)]
        L.ezqo_quantize.restype = I64
        L.ezqo_dequantize.argtypes = [I64, I64, I32, P, P, P, I64, P]
        L.ezqo_reconstruction_error.argtypes = [P, P, I64, I64, P, I64]
        L.ezqo_reconstruction_error.restype = D
        L.ezqo_packed_size.argtypes = [I64, I32]
        L.ezqo_packed_size.restype = I64
        L.ezqo_pack_levels.argtypes = [P, I64, I32, P]
        L.ezqo_unpack_levels.argtypes = [P, I64, I64, I32, P]
        L.ezqo_gemv_f64.argtypes = [P, I64, I64, P, I32, P]
        _lib = L
    return _lib


def cfg_c(cfg) -> OConfig:
    return OConfig(cfg.bits, cfg.sigma_n, cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.steps,
                   1 if getattr(cfg, "select", "best") == "fixed" else 0, cfg.select_step, 0,
                   getattr(cfg, "seed", 0))


def _p(a):
    return None if a is None else a.ctypes.data


def gaussian(rows, cols, seed, scale=1.0) -> np.ndarray:
    out = np.empty((rows, cols), np.float32)
    lib().ezqo_gaussian(_p(out), out.size, seed, scale)
    return out


def plant_outliers(W, count, lo, hi, seed):
    if lib().ezqo_plant_outliers(_p(W), W.size, count, lo, hi, seed) != 0:
        raise MemoryError("plant_outliers")
    return W


def tensor_stats(W) -> dict:
    m, s, a = C.c_double(), C.c_double(), C.c_double()
    lib().ezqo_tensor_stats(_p(np.ascontiguousarray(W, np.float32)), W.size, C.byref(m), C.byref(s),
                            C.byref(a))
    return {"mean": m.value, "stddev": s.value, "max_abs": a.value, "count": W.size}


def detect_outliers(W, sigma_n):
    W = np.ascontiguousarray(W, np.float32)
    m, s = C.c_double(), C.c_double()
    n = lib().ezqo_detect_outliers(_p(W), W.shape[0], W.shape[1], sigma_n, None, C.byref(m), C.byref(s))
    out = np.zeros(n, OUTLIER_DTYPE)
    lib().ezqo_detect_outliers(_p(W), W.shape[0], W.shape[1], sigma_n, _p(out), C.byref(m), C.byref(s))
    return out, m.value, s.value


def quantize(W, cfg, mode="easyquant", threads=None) -> dict:
    W = np.ascontiguousarray(W, np.float32)
    rows, cols = W.shape
    c = cfg_c(cfg)
    packed = np.zeros(max(lib().ezqo_packed_size(W.size, cfg.bits), 1), np.uint8)
    scales = np.zeros(cols, np.float32)
    m, s, r, f = C.c_double(), C.c_double(), C.c_double(), C.c_double()
    th = threads or os.cpu_count() or 1
    cap = max(W.size // 16, 1)
    outl = np.zeros(cap, OUTLIER_DTYPE)
    n = lib().ezqo_quantize(_p(W), rows, cols, C.byref(c), MODES[mode], th, _p(packed), _p(scales),
                            _p(outl), cap, C.byref(m), C.byref(s), C.byref(r), C.byref(f))
    if n > cap:
        outl = np.zeros(n, OUTLIER_DTYPE)
        n = lib().ezqo_quantize(_p(W), rows, cols, C.byref(c), MODES[mode], th, _p(packed),
                                _p(scales), _p(outl), n, C.byref(m), C.byref(s), C.byref(r),
                                C.byref(f))
    if n == -1:
        raise ValueError("non-finite element")
    if n == -3:
        raise ValueError("invalid config")
    status = "invariant" if n == -2 else "ok"
    return {"packed": packed[:lib().ezqo_packed_size(W.size, cfg.bits)], "scales": scales,
            "outliers": outl[:max(n, 0)], "mean": m.value, "stddev": s.value,
            "rtn_error": r.value, "final_error": f.value, "status": status}


def dequantize(rows, cols, bits, packed, scales, outliers) -> np.ndarray:
    out = np.zeros((rows, cols), np.float32)
    o = np.ascontiguousarray(outliers, OUTLIER_DTYPE)
    rc = lib().ezqo_dequantize(rows, cols, bits, _p(np.ascontiguousarray(packed, np.uint8)),
                               _p(np.ascontiguousarray(scales, np.float32)), _p(o), o.size, _p(out))
    if rc != 0:
        raise ValueError("outlier coordinate out of range")
    return out


def eval_dense(x, s, bits):
    x = np.ascontiguousarray(x, np.float32)
    e, g = C.c_double(), C.c_double()
    lmin, lmax = 1 - (1 << (bits - 1)), 1 << (bits - 1)
    lib().ezqo_eval_dense(_p(x), x.size, s, lmin, lmax, C.byref(e), C.byref(g))
    return e.value, g.value


def optimize_channel(v, cfg, keep_trace=False) -> dict:
    v = np.ascontiguousarray(v, np.float32)
    c = cfg_c(cfg)
    ie, fe = C.c_double(), C.c_double()
    bs = C.c_int()
    n = max(cfg.steps, 0) + 1
    ts = np.zeros(n) if keep_trace else None
    te = np.zeros(n) if keep_trace else None
    sc = lib().ezqo_optimize_channel(_p(v), v.size, C.byref(c), C.byref(ie), C.byref(fe),
                                     C.byref(bs), _p(ts), _p(te))
    return {"scale": sc, "initial_error": ie.value, "final_error": fe.value,
            "best_step": bs.value, "trace_scale": ts, "trace_error": te}


def brute_force(v, cfg, grid_points=2000):
    v = np.ascontiguousarray(v, np.float32)
    c = cfg_c(cfg)
    s, e = C.c_double(), C.c_double()
    lib().ezqo_brute_force(_p(v), v.size, C.byref(c), grid_points, C.byref(s), C.byref(e))
    return s.value, e.value


def adam_step(state, scale, grad, cfg):
    m, v, t = C.c_double(state["m"]), C.c_double(state["v"]), C.c_int64(state["t"])
    c = cfg_c(cfg)
    r = lib().ezqo_adam_step(C.byref(m), C.byref(v), C.byref(t), scale, grad, C.byref(c))
    state.update(m=m.value, v=v.value, t=t.value)
    return r


def level_of(x, inv, lmin, lmax):
    return lib().ezqo_level_of(x, inv, lmin, lmax)


def initial_scale(x, bits):
    x = np.ascontiguousarray(x, np.float32)
    return lib().ezqo_initial_scale(_p(x), x.size, bits)


def pack_levels(levels, bits):
    lv = np.ascontiguousarray(levels, np.int16)
    out = np.zeros(lib().ezqo_packed_size(lv.size, bits), np.uint8)
    if lib().ezqo_pack_levels(_p(lv), lv.size, bits, _p(out)) != 0:
        raise ValueError("level out of range")
    return out


def unpack_levels(b, count, bits):
    b = np.ascontiguousarray(b, np.uint8)
    out = np.zeros(count, np.int16)
    rc = lib().ezqo_unpack_levels(_p(b), b.size, count, bits, _p(out))
    if rc != 0:
        raise ValueError("bad packed buffer")
    return out


def reconstruction_error(a, b, skip=None):
    s = None if skip is None else np.ascontiguousarray(skip, OUTLIER_DTYPE)
    return lib().ezqo_reconstruction_error(_p(np.ascontiguousarray(a, np.float32)),
                                           _p(np.ascontiguousarray(b, np.float32)), a.shape[0],
                                           a.shape[1], _p(s), 0 if s is None else s.size)


def gemv_f64(What, x):
    What = np.ascontiguousarray(What, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    batch = x.shape[0]
    y = np.zeros((batch, What.shape[1]), np.float64)
    lib().ezqo_gemv_f64(_p(What), What.shape[0], What.shape[1], _p(x), batch, _p(y))
    return y


# ---- dense 3-bit stream (test restatement of include/ezquant_c.h's layout) --
# The reference has no dense 3-bit format (it stores k = 3 one offset byte per
# level, rtn.cpp:119-147); this is the plain definition the device codec is
# checked against: offset e at bits 3e..3e+2 of a little-endian bit stream.
def dense3_size(count):
    return 0 if count <= 0 else 3 * ((count + 7) // 8)


def dense3_pack(offsets):
    o = np.ascontiguousarray(offsets, np.uint8).ravel()
    if o.size and int(o.max()) > 7:
        raise ValueError("offset exceeds level span 7")
    n = o.size
    g = np.zeros(((n + 7) // 8) * 8, np.uint32)
    g[:n] = o
    g = g.reshape(-1, 8)
    word = np.zeros(g.shape[0], np.uint32)
    for i in range(8):
        word |= g[:, i] << np.uint32(3 * i)
    out = np.stack([(word >> np.uint32(8 * b)) & np.uint32(0xFF) for b in range(3)], axis=1)
    return out.astype(np.uint8).ravel()


def dense3_unpack(stream, count):
    s = np.ascontiguousarray(stream, np.uint8).ravel()[: dense3_size(count)].reshape(-1, 3).astype(np.uint32)
    word = s[:, 0] | (s[:, 1] << np.uint32(8)) | (s[:, 2] << np.uint32(16))
    out = np.stack([(word >> np.uint32(3 * i)) & np.uint32(7) for i in range(8)], axis=1)
    return out.astype(np.uint8).ravel()[:count]

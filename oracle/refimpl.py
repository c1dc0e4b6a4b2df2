"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/_ref/libezq_ref.so.

libezq_ref.so is the UNMODIFIED reference library (EasyQuant `ezquant`,
/root/reference/proj) compiled out-of-tree by oracle/Makefile plus the C shim
oracle/ref_capi.cpp. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may use it, and only as the checker or
the timed CPU baseline -- never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libezq_ref.so")
OUTLIER_DTYPE = np.dtype([("row", "<u4"), ("col", "<u4"), ("value", "<f4")])
MODES = {"easyquant": 0, "rtn": 1, "outliers-only": 2}


class RefConfig(C.Structure):
    _fields_ = [("bits", C.c_int32), ("sigma_n", C.c_float), ("lr", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("steps", C.c_int32), ("select", C.c_int32), ("select_step", C.c_int32),
                ("pad", C.c_int32), ("seed", C.c_uint64)]


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[ref {code}] {msg}")
        self.code, self.msg = code, msg


_lib = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {REF_SO}")
        L = C.CDLL(REF_SO)
        P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int, C.c_double
        L.ref_last_error.restype = C.c_char_p
        L.ref_gaussian.argtypes = [P, I64, C.c_uint64, D]
        L.ref_plant_outliers.argtypes = [P, I64, I64, D, D, C.c_uint64]
        L.ref_tensor_stats.argtypes = [P, I64, I64, I32, P, C.POINTER(I64)]
        L.ref_detect_outliers.argtypes = [P, I64, I64, C.POINTER(RefConfig), I32, C.POINTER(I64),
                                          P, P, P, C.POINTER(D), C.POINTER(D)]
        L.ref_quantize.argtypes = [P, I64, I64, C.POINTER(RefConfig), I32, I32, C.POINTER(C.c_int)]
        L.ref_quantize.restype = P
        L.ref_q_free.argtypes = [P]
        L.ref_q_packed.argtypes = [P, P]
        L.ref_q_packed.restype = I64
        L.ref_q_scales.argtypes = [P, P]
        L.ref_q_outliers.argtypes = [P, P, P, P]
        L.ref_q_outliers.restype = I64
        L.ref_q_meta.argtypes = [P, P, C.POINTER(C.c_float), C.POINTER(C.c_int)]
        L.ref_q_make.argtypes = [I64, I64, I32, P, I64, P, I64, P, P, P, D, D, C.c_float]
        L.ref_q_make.restype = P
        L.ref_dequantize.argtypes = [P, P, I32]
        L.ref_encode.argtypes = [P, P]
        L.ref_encode.restype = I64
        L.ref_decode.argtypes = [P, I64, C.POINTER(C.c_int), C.POINTER(C.c_uint64)]
        L.ref_decode.restype = P
        L.ref_quantize_model.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(RefConfig), C.c_int,
                                         C.c_int, C.POINTER(C.c_int)]
        L.ref_dequantize_model.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_int)]
        L.ref_sigma_sweep.argtypes = [C.c_char_p, C.POINTER(RefConfig), P, C.c_int, C.c_int,
                                      C.c_char_p, I64]
        L.ref_channel_eval.argtypes = [P, I64, P, I64, D, C.POINTER(RefConfig), C.POINTER(D),
                                       C.POINTER(D)]
        L.ref_adam_step.argtypes = [C.POINTER(D), C.POINTER(D), C.POINTER(I64), D, D,
                                    C.POINTER(RefConfig)]
        L.ref_adam_step.restype = D
        L.ref_optimize_channel.argtypes = [P, I64, P, I64, C.POINTER(RefConfig), I32,
                                           C.POINTER(C.c_float), C.POINTER(D), C.POINTER(D),
                                           C.POINTER(C.c_int), C.POINTER(D), C.POINTER(D),
                                           C.POINTER(C.c_int), P, P, P]
        L.ref_brute_force.argtypes = [P, I64, P, I64, C.POINTER(RefConfig), I32, C.POINTER(D),
                                      C.POINTER(D)]
        L.ref_initial_scale.argtypes = [P, I64, C.POINTER(RefConfig)]
        L.ref_initial_scale.restype = D
        L.ref_quantize_channel.argtypes = [P, I64, D, C.POINTER(RefConfig), P]
        L.ref_dequantize_channel.argtypes = [P, I64, I32, D, P]
        L.ref_packed_size.argtypes = [I64, I32]
        L.ref_packed_size.restype = I64
        L.ref_pack_levels.argtypes = [P, I64, I32, P]
        L.ref_unpack_levels.argtypes = [P, I64, I64, I32, P]
        L.ref_reconstruction_error.argtypes = [P, P, I64, I64, P, P, I64, I32, C.POINTER(D)]
        L.ref_set_threads.argtypes = [I32]
        L.ref_max_threads.restype = I32
        _lib = L
    return _lib


def cfg_c(cfg) -> RefConfig:
    """Accepts any object with the Config fields (paper_2403_02775_b200.native.Config)."""
    sel = 1 if getattr(cfg, "select", "best") == "fixed" else 0
    return RefConfig(cfg.bits, cfg.sigma_n, cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.steps, sel,
                     cfg.select_step, 0, getattr(cfg, "seed", 0))


def _check(code):
    if code != 0:
        raise RefError(code, lib().ref_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data


def set_threads(n: int):
    lib().ref_set_threads(n)


def max_threads() -> int:
    return lib().ref_max_threads()


# ---- synthetic inputs (reference Rng, rng.hpp) -----------------------------
def gaussian(rows: int, cols: int, seed: int, scale: float = 1.0) -> np.ndarray:
    out = np.empty((rows, cols), np.float32)
    lib().ref_gaussian(out.ctypes.data, out.size, seed, scale)
    return out


def plant_outliers(W: np.ndarray, count: int, lo: float, hi: float, seed: int) -> np.ndarray:
    lib().ref_plant_outliers(W.ctypes.data, W.size, count, lo, hi, seed)
    return W


# ---- API mirrors -------------------------------------------------------------
def tensor_stats(W, serial=False):
    out = np.zeros(3, np.float64)
    cnt = C.c_int64(0)
    _check(lib().ref_tensor_stats(_p(W), W.shape[0], W.shape[1], int(serial), out.ctypes.data,
                                  C.byref(cnt)))
    return {"mean": out[0], "stddev": out[1], "max_abs": out[2], "count": cnt.value}


def detect_outliers(W, cfg, serial=False):
    c = cfg_c(cfg)
    n = C.c_int64(0)
    m, s = C.c_double(0), C.c_double(0)
    _check(lib().ref_detect_outliers(_p(W), W.shape[0], W.shape[1], C.byref(c), int(serial),
                                     C.byref(n), None, None, None, C.byref(m), C.byref(s)))
    r = np.zeros(n.value, np.uint32)
    cc = np.zeros(n.value, np.uint32)
    v = np.zeros(n.value, np.float32)
    _check(lib().ref_detect_outliers(_p(W), W.shape[0], W.shape[1], C.byref(c), int(serial),
                                     C.byref(n), _p(r), _p(cc), _p(v), C.byref(m), C.byref(s)))
    out = np.zeros(n.value, OUTLIER_DTYPE)
    out["row"], out["col"], out["value"] = r, cc, v
    return out, m.value, s.value


class RefQuantized:
    def __init__(self, h):
        self.h = h
        L = lib()
        self.packed = np.zeros(L.ref_q_packed(h, None), np.uint8)
        L.ref_q_packed(h, _p(self.packed))
        meta = np.zeros(4, np.float64)
        sig = C.c_float(0)
        bits = C.c_int(0)
        L.ref_q_meta(h, meta.ctypes.data, C.byref(sig), C.byref(bits))
        self.mean, self.stddev, self.rtn_error, self.final_error = meta
        self.sigma_n, self.bits = sig.value, bits.value
        n = L.ref_q_outliers(h, None, None, None)
        r, c, v = np.zeros(n, np.uint32), np.zeros(n, np.uint32), np.zeros(n, np.float32)
        L.ref_q_outliers(h, _p(r), _p(c), _p(v))
        self.outliers = np.zeros(n, OUTLIER_DTYPE)
        self.outliers["row"], self.outliers["col"], self.outliers["value"] = r, c, v

    def load_scales(self, cols):
        self.scales = np.zeros(cols, np.float32)
        lib().ref_q_scales(self.h, _p(self.scales))
        return self

    def dequantize(self, rows, cols, serial=False):
        out = np.zeros((rows, cols), np.float32)
        _check(lib().ref_dequantize(self.h, _p(out), int(serial)))
        return out

    def encode(self) -> bytes:
        n = lib().ref_encode(self.h, None)
        b = np.zeros(n, np.uint8)
        lib().ref_encode(self.h, _p(b))
        return b.tobytes()

    def __del__(self):
        try:
            lib().ref_q_free(self.h)
        except Exception:
            pass


def quantize(W, cfg, mode="easyquant", serial=False) -> RefQuantized:
    c = cfg_c(cfg)
    st = C.c_int(0)
    h = lib().ref_quantize(_p(W), W.shape[0], W.shape[1], C.byref(c), MODES[mode], int(serial),
                           C.byref(st))
    if not h:
        raise RefError(st.value, lib().ref_last_error().decode())
    q = RefQuantized(h)
    q.rows, q.cols = W.shape
    return q.load_scales(W.shape[1])


def make_quantized(rows, cols, bits, packed, scales, outliers, mean=0.0, stddev=0.0, sigma_n=0.0):
    packed = np.ascontiguousarray(packed, np.uint8)
    scales = np.ascontiguousarray(scales, np.float32)
    r = np.ascontiguousarray(outliers["row"], np.uint32)
    c = np.ascontiguousarray(outliers["col"], np.uint32)
    v = np.ascontiguousarray(outliers["value"], np.float32)
    h = lib().ref_q_make(rows, cols, bits, _p(packed), packed.size, _p(scales), len(r), _p(r),
                         _p(c), _p(v), mean, stddev, sigma_n)
    q = RefQuantized(h)
    q.rows, q.cols = rows, cols
    q.scales = scales
    return q


def decode(b: bytes):
    arr = np.frombuffer(b, np.uint8).copy()
    st = C.c_int(0)
    off = C.c_uint64(0)
    h = lib().ref_decode(_p(arr) if arr.size else None, arr.size, C.byref(st), C.byref(off))
    if not h:
        e = RefError(st.value, lib().ref_last_error().decode())
        e.offset = off.value
        raise e
    return RefQuantized(h)


def channel_eval(x, mask, s, cfg):
    x = np.ascontiguousarray(x, np.float32)
    m = None if mask is None else np.ascontiguousarray(mask, np.uint32)
    c = cfg_c(cfg)
    e, g = C.c_double(0), C.c_double(0)
    _check(lib().ref_channel_eval(_p(x), x.size, _p(m), 0 if m is None else m.size, s, C.byref(c),
                                  C.byref(e), C.byref(g)))
    return e.value, g.value


def optimize_channel(x, mask, cfg, keep_trace=False):
    x = np.ascontiguousarray(x, np.float32)
    m = None if mask is None else np.ascontiguousarray(mask, np.uint32)
    c = cfg_c(cfg)
    n = max(cfg.steps, 0) + 1
    ts, sc, er = np.zeros(n, np.int32), np.zeros(n), np.zeros(n)
    scale = C.c_float(0)
    ie, fe, bs, be = C.c_double(0), C.c_double(0), C.c_double(0), C.c_double(0)
    bstep, ntr = C.c_int(0), C.c_int(0)
    _check(lib().ref_optimize_channel(_p(x), x.size, _p(m), 0 if m is None else m.size, C.byref(c),
                                      int(keep_trace), C.byref(scale), C.byref(ie), C.byref(fe),
                                      C.byref(bstep), C.byref(bs), C.byref(be), C.byref(ntr),
                                      _p(ts), _p(sc), _p(er)))
    k = ntr.value
    return {"scale": scale.value, "initial_error": ie.value, "final_error": fe.value,
            "best_step": bstep.value, "best_scale": bs.value, "best_error": be.value,
            "trace_step": ts[:k], "trace_scale": sc[:k], "trace_error": er[:k]}


def brute_force_scale(x, mask, cfg, grid_points=2000):
    x = np.ascontiguousarray(x, np.float32)
    m = None if mask is None else np.ascontiguousarray(mask, np.uint32)
    c = cfg_c(cfg)
    s, e = C.c_double(0), C.c_double(0)
    _check(lib().ref_brute_force(_p(x), x.size, _p(m), 0 if m is None else m.size, C.byref(c),
                                 grid_points, C.byref(s), C.byref(e)))
    return s.value, e.value


def quantize_channel(x, s, cfg):
    x = np.ascontiguousarray(x, np.float32)
    out = np.zeros(x.size, np.int16)
    c = cfg_c(cfg)
    _check(lib().ref_quantize_channel(_p(x), x.size, s, C.byref(c), _p(out)))
    return out


def initial_scale(x, cfg):
    x = np.ascontiguousarray(x, np.float32)
    c = cfg_c(cfg)
    return lib().ref_initial_scale(_p(x), x.size, C.byref(c))


def adam_step(state, scale, grad, cfg):
    m, v, t = C.c_double(state["m"]), C.c_double(state["v"]), C.c_int64(state["t"])
    c = cfg_c(cfg)
    r = lib().ref_adam_step(C.byref(m), C.byref(v), C.byref(t), scale, grad, C.byref(c))
    state.update(m=m.value, v=v.value, t=t.value)
    return r


def pack_levels(levels, bits):
    lv = np.ascontiguousarray(levels, np.int16)
    out = np.zeros(lib().ref_packed_size(lv.size, bits), np.uint8)
    _check(lib().ref_pack_levels(_p(lv), lv.size, bits, _p(out)))
    return out


def unpack_levels(b, count, bits):
    b = np.ascontiguousarray(b, np.uint8)
    out = np.zeros(count, np.int16)
    _check(lib().ref_unpack_levels(_p(b), b.size, count, bits, _p(out)))
    return out


def reconstruction_error(a, b, skip=None, serial=False):
    r = c = None
    n = 0
    if skip is not None:
        r = np.ascontiguousarray(skip["row"], np.uint32)
        c = np.ascontiguousarray(skip["col"], np.uint32)
        n = len(skip)
    out = C.c_double(0)
    _check(lib().ref_reconstruction_error(_p(a), _p(b), a.shape[0], a.shape[1], _p(r), _p(c), n,
                                          int(serial), C.byref(out)))
    return out.value


def quantize_model(manifest: str, out_dir: str, cfg, mode="easyquant", workers=4) -> int:
    """model.hpp quantize_model of the compiled reference; returns failures."""
    c = cfg_c(cfg)
    f = C.c_int(0)
    _check(lib().ref_quantize_model(manifest.encode(), out_dir.encode(), C.byref(c), MODES[mode],
                                    workers, C.byref(f)))
    return f.value


def dequantize_model(in_dir: str, out_dir: str, workers=4) -> int:
    f = C.c_int(0)
    _check(lib().ref_dequantize_model(in_dir.encode(), out_dir.encode(), workers, C.byref(f)))
    return f.value


def sigma_sweep(manifest: str, cfg, sigmas, workers=4) -> str:
    """report.hpp sigma_sweep of the compiled reference, as sweep_to_json text."""
    c = cfg_c(cfg)
    sg = np.ascontiguousarray(sigmas, np.float32)
    buf = C.create_string_buffer(1 << 20)
    _check(lib().ref_sigma_sweep(manifest.encode(), C.byref(c), _p(sg), sg.size, workers, buf,
                                 1 << 20))
    return buf.value.decode()

"""ctypes binding of the B200 engine's C-ABI (include/ezquant_c.h).

This is the Python face of the drop-in boundary: the same entry points a
reference integrator would bind. Arrays are numpy (host) or
torch CUDA tensors (device, passed by data_ptr()). There is no CPU fallback:
if libezq_b200.so is missing or no CUDA device exists, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "_lib")
LIB_PATH = os.environ.get("EZQ_LIB") or os.path.join(LIB_DIR, "libezq_b200.so")  # EZQ_LIB: A/B builds (dev aid)

OK, INVALID_ARGUMENT, INVARIANT, IO_FAILURE, IO_FORMAT, IO_VERSION = 0, 1, 2, 3, 4, 5
CUDA_ERROR, NO_DEVICE, OOM = 10, 11, 12
MEM_HOST, MEM_DEVICE = 0, 1
MODES = {"easyquant": 0, "rtn": 1, "outliers-only": 2}
SELECT_BEST, SELECT_FIXED = 0, 1


class EzqError(RuntimeError):
    def __init__(self, code: int, msg: str, index: int):
        super().__init__(f"[ezq {code}] {msg}")
        self.code, self.msg, self.index = code, msg, index


class InvalidArgument(EzqError, ValueError):
    pass


class InvariantError(EzqError):
    pass


class IoError(EzqError):
    pass


class CConfig(C.Structure):
    _fields_ = [("bits", C.c_int32), ("sigma_n", C.c_float), ("lr", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("steps", C.c_int32), ("select", C.c_int32), ("select_step", C.c_int32),
                ("reserved", C.c_int32), ("seed", C.c_uint64)]


class CStats(C.Structure):
    _fields_ = [("mean", C.c_double), ("stddev", C.c_double), ("max_abs", C.c_double),
                ("count", C.c_int64)]


class COutlier(C.Structure):
    _fields_ = [("row", C.c_uint32), ("col", C.c_uint32), ("value", C.c_float)]


OUTLIER_DTYPE = np.dtype([("row", "<u4"), ("col", "<u4"), ("value", "<f4")])


class CQWeight(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("bits", C.c_int32), ("mem", C.c_int32),
                ("packed_bytes", C.c_int64), ("packed", C.POINTER(C.c_uint8)),
                ("scales", C.POINTER(C.c_float)), ("n_outliers", C.c_int64),
                ("outliers", C.POINTER(COutlier)), ("mean", C.c_double), ("stddev", C.c_double),
                ("sigma_n", C.c_float), ("has_errors", C.c_int32), ("rtn_error", C.c_double),
                ("final_error", C.c_double), ("owned", C.c_int32), ("reserved", C.c_int32)]


class COptResult(C.Structure):
    _fields_ = [("scale", C.c_float), ("best_step", C.c_int32), ("initial_error", C.c_double),
                ("final_error", C.c_double), ("best_scale", C.c_double),
                ("best_error", C.c_double), ("n_trace", C.c_int32), ("reserved", C.c_int32)]


@dataclass
class Config:
    """QuantConfig (types.hpp:37-54) with the reference defaults."""
    bits: int = 4
    sigma_n: float = 3.0
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    steps: int = 200
    select: str = "best"          # "best" | "fixed"
    select_step: int = 100
    seed: int = 0

    def to_c(self) -> CConfig:
        return CConfig(self.bits, self.sigma_n, self.lr, self.beta1, self.beta2, self.eps,
                       self.steps, SELECT_FIXED if self.select == "fixed" else SELECT_BEST,
                       self.select_step, 0, self.seed)

    @property
    def level_min(self) -> int:
        return -(1 << (self.bits - 1)) + 1

    @property
    def level_max(self) -> int:
        return 1 << (self.bits - 1)


@dataclass
class QuantizedWeight:
    """Host copy of QuantizedWeight (types.hpp:103-113)."""
    rows: int
    cols: int
    bits: int
    packed: np.ndarray                  # uint8
    scales: np.ndarray                  # float32 [cols]
    outliers: np.ndarray                # OUTLIER_DTYPE, sorted by (row, col)
    mean: float = 0.0
    stddev: float = 0.0
    sigma_n: float = 0.0
    rtn_error: Optional[float] = None
    final_error: Optional[float] = None
    _owner: object = field(default=None, repr=False, compare=False)

    def __getstate__(self):
        """Pickles as plain arrays: zero-copy views of library memory are
        copied and the owner handle (a ctypes pointer) is dropped."""
        d = dict(self.__dict__)
        for k in ("packed", "scales", "outliers"):
            d[k] = np.array(d[k], copy=True)
        d["_owner"] = None
        return d


class _OwnedBuffer:
    """Exposes `nbytes` of library memory at `addr` through the array
    interface and holds the owner: numpy arrays built on it keep the owner
    (and so the memory) alive for as long as any view exists."""

    def __init__(self, addr: int, nbytes: int, owner):
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (addr, False), "version": 3}
        self._owner = owner


def _owned_view(addr: int, count: int, dtype, owner) -> np.ndarray:
    dt = np.dtype(dtype)
    return np.asarray(_OwnedBuffer(addr, count * dt.itemsize, owner)).view(dt)


class _COwner:
    """Keeps a library-owned host ezq_qweight alive while numpy views of its
    arrays exist (zero-copy results); frees it with ezq_qweight_free."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            if self.ptr:
                lib().ezq_qweight_free(self.ptr)
        except Exception:
            pass


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"B200 engine not built: {LIB_PATH} missing (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int, C.c_double
        L.ezq_last_error.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_int64)]
        L.ezq_config_validate.argtypes = [C.POINTER(CConfig)]
        L.ezq_device_count.argtypes = [C.POINTER(C.c_int)]
        L.ezq_set_device.argtypes = [I32]
        L.ezq_version.restype = C.c_char_p
        L.ezq_kernel_launches.restype = I64
        L.ezq_tie_stats.argtypes = [C.POINTER(I64), C.POINTER(I64)]
        L.ezq_tensor_stats.argtypes = [P, I64, I64, I32, P, C.POINTER(CStats)]
        L.ezq_detect_outliers.argtypes = [P, I64, I64, C.POINTER(CConfig), I32, P,
                                          C.POINTER(C.POINTER(COutlier)), C.POINTER(I64),
                                          C.POINTER(D), C.POINTER(D)]
        L.ezq_quantize_tensor.argtypes = [P, I64, I64, C.POINTER(CConfig), I32, I32, I32, P,
                                          C.POINTER(C.POINTER(CQWeight))]
        L.ezq_quantize_batch.argtypes = [C.POINTER(P), C.POINTER(I64), C.POINTER(I64), I32,
                                         C.POINTER(CConfig), I32, I32, I32, P,
                                         C.POINTER(C.POINTER(CQWeight)), C.POINTER(C.c_int)]
        L.ezq_grid_oracle_batch.argtypes = [C.POINTER(P), C.POINTER(I64), C.POINTER(I64), I32,
                                            C.POINTER(CConfig), I32, I32, P, P, P, C.POINTER(C.c_int)]
        L.ezq_sigma_sweep_batch.argtypes = [C.POINTER(P), C.POINTER(I64), C.POINTER(I64), I32,
                                            C.POINTER(CConfig), I32, P, P, I32, P, P, P, C.POINTER(C.c_int)]
        L.ezq_dequantize_tensor.argtypes = [C.POINTER(CQWeight), P, I32, P]
        L.ezq_qweight_wrap.argtypes = [I64, I64, I32, P, I64, P, I64, P, I64, D, D, C.c_float,
                                       I32, C.POINTER(C.POINTER(CQWeight))]
        L.ezq_qweight_free.argtypes = [C.POINTER(CQWeight)]
        L.ezq_qweight_to_host.argtypes = [C.POINTER(CQWeight), C.POINTER(C.POINTER(CQWeight))]
        L.ezq_free.argtypes = [P]
        L.ezq_reconstruction_error.argtypes = [P, P, I64, I64, P, P, I64, I32, P, C.POINTER(D)]
        L.ezq_channel_eval.argtypes = [P, I64, P, I64, D, C.POINTER(CConfig), C.POINTER(D),
                                       C.POINTER(D)]
        L.ezq_optimize_channel.argtypes = [P, I64, P, I64, C.POINTER(CConfig), I32,
                                           C.POINTER(COptResult), P, P, P]
        L.ezq_brute_force_scale.argtypes = [P, I64, P, I64, C.POINTER(CConfig), I32,
                                            C.POINTER(D), C.POINTER(D)]
        L.ezq_quantize_channel.argtypes = [P, I64, D, C.POINTER(CConfig), P]
        L.ezq_initial_scale.argtypes = [P, I64, C.POINTER(CConfig)]
        L.ezq_initial_scale.restype = D
        L.ezq_adam_step.argtypes = [C.POINTER(D), C.POINTER(D), C.POINTER(I64), D, D,
                                    C.POINTER(CConfig), C.POINTER(D)]
        L.ezq_packed_size.argtypes = [I64, I32]
        L.ezq_packed_size.restype = I64
        L.ezq_pack_levels.argtypes = [P, I64, I32, P]
        L.ezq_unpack_levels.argtypes = [P, I64, I64, I32, P]
        L.ezq_dequantize_channel.argtypes = [P, I64, D, P]
        L.ezq_gemv_prepare.argtypes = [C.POINTER(CQWeight), P, C.POINTER(P)]
        L.ezq_gemv_prepare_ex.argtypes = [C.POINTER(CQWeight), I32, P, C.POINTER(P)]
        L.ezq_gemv.argtypes = [P, P, I32, I32, P, P]
        L.ezq_gemv_plan_free.argtypes = [P]
        L.ezq_dense3_size.argtypes = [I64]
        L.ezq_dense3_size.restype = I64
        L.ezq_pack_dense3.argtypes = [P, I64, P, I32, P]
        L.ezq_unpack_dense3.argtypes = [P, I64, P, I32, P]
        L.ezq_dequantize_dense3.argtypes = [C.POINTER(CQWeight), P, P, I32, P]
        L.ezq_gemv_prepare_dense3.argtypes = [C.POINTER(CQWeight), P, I32, P, C.POINTER(P)]
        L.ezq_profile_enable.argtypes = [I32]
        L.ezq_profile_read.argtypes = [C.c_char_p, C.POINTER(D), C.POINTER(I64), C.POINTER(D)]
        L.ezq_measure_fp64_peak.argtypes = [C.POINTER(D)]
        L.ezq_encode_quantized.argtypes = [C.POINTER(CQWeight), C.POINTER(C.POINTER(C.c_uint8)),
                                           C.POINTER(I64)]
        L.ezq_decode_quantized.argtypes = [P, I64, C.POINTER(C.POINTER(CQWeight))]
        _lib = L
    return _lib


def _raise(code: int):
    buf = C.create_string_buffer(2048)
    idx = C.c_int64(-1)
    lib().ezq_last_error(buf, 2048, C.byref(idx))
    msg = buf.value.decode()
    cls = {INVALID_ARGUMENT: InvalidArgument, INVARIANT: InvariantError, IO_FAILURE: IoError,
           IO_FORMAT: IoError, IO_VERSION: IoError}.get(code, EzqError)
    raise cls(code, msg, idx.value)


def check(code: int):
    if code != OK:
        _raise(code)


def _as_f32(W):
    """A float32 row-major matrix the C-ABI can read: numpy inputs are made
    contiguous float32 (a copy when needed); torch inputs must be float32 and
    contiguous (a transposed view or a 16-bit tensor would be read as the
    wrong bytes) and are converted with .contiguous().float() otherwise."""
    if isinstance(W, np.ndarray):
        return np.ascontiguousarray(W, dtype=np.float32)
    import torch
    if W.dtype != torch.float32 or not W.is_contiguous():
        W = W.contiguous().to(torch.float32)
    return W


def _ptr(a) -> Optional[int]:
    """Address of a numpy array or torch tensor (None for None)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _mem(a) -> int:
    return MEM_HOST if isinstance(a, np.ndarray) else (MEM_DEVICE if a.is_cuda else MEM_HOST)


def _stream(stream, *tensors) -> Optional[int]:
    """Explicit stream, else torch's current stream when any argument is a
    torch CUDA tensor (so library work is ordered after the producer of the
    inputs and before their consumers), else the library's own stream."""
    if stream is not None:
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    for t in tensors:
        if t is not None and not isinstance(t, np.ndarray) and getattr(t, "is_cuda", False):
            import torch
            h = torch.cuda.current_stream(t.device).cuda_stream
            return h if h else 1  # torch's legacy default stream -> cudaStreamLegacy
    return None


def device_count() -> int:
    n = C.c_int(0)
    lib().ezq_device_count(C.byref(n))
    return n.value


def set_device(d: int):
    check(lib().ezq_set_device(d))


def kernel_launches() -> int:
    return int(lib().ezq_kernel_launches())


def tie_stats() -> tuple:
    """Cumulative (resolved, fallback) near-tie columns (ezq_tie_stats)."""
    a, b = C.c_int64(0), C.c_int64(0)
    check(lib().ezq_tie_stats(C.byref(a), C.byref(b)))
    return int(a.value), int(b.value)


def profile_enable(on: bool = True):
    check(lib().ezq_profile_enable(int(on)))


def profile_read(family: str) -> dict:
    ms, n, w = C.c_double(), C.c_int64(), C.c_double()
    check(lib().ezq_profile_read(family.encode(), C.byref(ms), C.byref(n), C.byref(w)))
    return {"ms": ms.value, "launches": n.value, "work": w.value}


def measure_fp64_peak() -> float:
    t = C.c_double()
    check(lib().ezq_measure_fp64_peak(C.byref(t)))
    return t.value


def config_validate(cfg: Config):
    c = cfg.to_c()
    check(lib().ezq_config_validate(C.byref(c)))


# ---- tensor-scale ---------------------------------------------------------
def tensor_stats(W, stream=None) -> dict:
    """stats.hpp:14 -> {mean, stddev, max_abs, count}."""
    W = _as_f32(W)
    rows, cols = W.shape
    st = CStats()
    check(lib().ezq_tensor_stats(_ptr(W), rows, cols, _mem(W), _stream(stream, W), C.byref(st)))
    return {"mean": st.mean, "stddev": st.stddev, "max_abs": st.max_abs, "count": st.count}


def detect_outliers(W, cfg: Config, stream=None):
    """outliers.hpp:15 -> (entries[OUTLIER_DTYPE], mean, stddev)."""
    W = _as_f32(W)
    rows, cols = W.shape
    c = cfg.to_c()
    e = C.POINTER(COutlier)()
    n = C.c_int64(0)
    mean, std = C.c_double(0), C.c_double(0)
    check(lib().ezq_detect_outliers(_ptr(W), rows, cols, C.byref(c), _mem(W), _stream(stream, W),
                                    C.byref(e), C.byref(n), C.byref(mean), C.byref(std)))
    out = np.zeros(n.value, dtype=OUTLIER_DTYPE)
    if n.value:
        C.memmove(out.ctypes.data, e, n.value * 12)
        lib().ezq_free(e)
    return out, mean.value, std.value


def _from_c(q: CQWeight, owner=None) -> QuantizedWeight:
    """Host artifact -> QuantizedWeight. With `owner` (a _COwner of the C
    struct) the arrays are zero-copy views kept alive by the owner; without it
    they are copied."""
    assert q.mem == MEM_HOST

    def arr(ptr, count, dtype):
        if not count:
            return np.zeros(0, dtype)
        addr = C.cast(ptr, C.c_void_p).value
        if owner is not None:
            return _owned_view(addr, count, dtype, owner)
        return _owned_view(addr, count, dtype, None).copy()

    packed = arr(q.packed, q.packed_bytes, np.uint8)
    scales = arr(q.scales, q.cols, np.float32)
    outl = arr(q.outliers, q.n_outliers, OUTLIER_DTYPE)
    return QuantizedWeight(q.rows, q.cols, q.bits, packed, scales, outl, q.mean, q.stddev,
                           q.sigma_n, q.rtn_error if q.has_errors else None,
                           q.final_error if q.has_errors else None, owner)


def quantize_tensor(W, cfg: Config, mode: str = "easyquant", stream=None) -> QuantizedWeight:
    """pipeline.hpp:33 -- host copy of the artifact (device work inside)."""
    W = _as_f32(W)
    rows, cols = W.shape
    c = cfg.to_c()
    q = C.POINTER(CQWeight)()
    check(lib().ezq_quantize_tensor(_ptr(W), rows, cols, C.byref(c), MODES[mode], _mem(W),
                                    MEM_HOST, _stream(stream, W), C.byref(q)))
    try:
        return _from_c(q.contents)
    finally:
        lib().ezq_qweight_free(q)


class DeviceBatch:
    """Device-resident outputs of ezq_quantize_batch (freed on close())."""

    def __init__(self, ptrs):
        self.ptrs = ptrs

    def __len__(self):
        return len(self.ptrs)

    def __getitem__(self, i) -> CQWeight:
        return self.ptrs[i].contents

    def to_host(self, i) -> "QuantizedWeight":
        h = C.POINTER(CQWeight)()
        check(lib().ezq_qweight_to_host(self.ptrs[i], C.byref(h)))
        try:
            return _from_c(h.contents)
        finally:
            lib().ezq_qweight_free(h)

    def dequantize_into(self, i, out, stream=None):
        """ezq_dequantize_tensor of entry i into `out` (torch CUDA tensor or numpy)."""
        check(lib().ezq_dequantize_tensor(self.ptrs[i], _ptr(out), _mem(out), _stream(stream, out)))
        return out

    def dequantize_dense3_into(self, i, dense, out, stream=None):
        """ezq_dequantize_dense3 of entry i (3-bit) from a device dense stream."""
        check(lib().ezq_dequantize_dense3(self.ptrs[i], _ptr(dense), _ptr(out), _mem(out), _stream(stream, out)))
        return out

    def close(self):
        for p in self.ptrs:
            if p:
                lib().ezq_qweight_free(p)
        self.ptrs = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def quantize_batch(Ws: Sequence, cfg: Config, mode: str = "easyquant", out_mem: int = MEM_HOST,
                   stream=None):
    """ezq_quantize_batch: list of QuantizedWeight (host) or a DeviceBatch."""
    Ws = [_as_f32(w) for w in Ws]
    n = len(Ws)
    if n and len({_mem(w) for w in Ws}) != 1:
        raise ValueError("quantize_batch: every tensor must live in the same memory (all host or all device)")
    ptrs = (C.c_void_p * n)(*[_ptr(w) for w in Ws])
    rows = (C.c_int64 * n)(*[w.shape[0] for w in Ws])
    cols = (C.c_int64 * n)(*[w.shape[1] for w in Ws])
    outs = (C.POINTER(CQWeight) * n)()
    failed = C.c_int(-1)
    c = cfg.to_c()
    check(lib().ezq_quantize_batch(ptrs, rows, cols, n, C.byref(c), MODES[mode], _mem(Ws[0]),
                                   out_mem, _stream(stream, Ws[0]), outs, C.byref(failed)))
    if out_mem == MEM_DEVICE:
        return DeviceBatch(list(outs))
    return [_from_c(p.contents, _COwner(p)) for p in outs]


class GemvPlan:
    """ezq_gemv_prepare / ezq_gemv over a device-resident artifact (a
    DeviceBatch entry). x: torch CUDA tensor [batch, rows] (f32/bf16/f16)."""

    DTYPES = {"torch.float32": 0, "torch.bfloat16": 1, "torch.float16": 2}
    OUTLIER_DTYPES = {"float32": 0, "float16": 1}

    def __init__(self, batch: "DeviceBatch", i: int, stream=None, outlier_dtype: str = "float32"):
        self._keep = batch
        self.rows, self.cols = batch[i].rows, batch[i].cols
        self.p = C.c_void_p()
        check(lib().ezq_gemv_prepare_ex(batch.ptrs[i], self.OUTLIER_DTYPES[outlier_dtype], _stream(stream),
                                        C.byref(self.p)))
        self.stream = stream

    def __call__(self, x, y=None, stream=None):
        import torch
        if y is None:
            y = torch.empty((x.shape[0], self.cols), dtype=torch.float32, device=x.device)
        check(lib().ezq_gemv(self.p, x.data_ptr(), self.DTYPES[str(x.dtype)], x.shape[0],
                             y.data_ptr(), _stream(stream or self.stream, x)))
        return y

    def close(self):
        if self.p:
            lib().ezq_gemv_plan_free(self.p)
            self.p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dequantize(q: QuantizedWeight, out=None, stream=None) -> np.ndarray:
    """pipeline.hpp:41 dequantize_tensor for a host artifact."""
    outl = np.ascontiguousarray(q.outliers, dtype=OUTLIER_DTYPE)
    w = C.POINTER(CQWeight)()
    packed = np.ascontiguousarray(q.packed, dtype=np.uint8)
    scales = np.ascontiguousarray(q.scales, dtype=np.float32)
    check(lib().ezq_qweight_wrap(q.rows, q.cols, q.bits, _ptr(packed), packed.size, _ptr(scales),
                                 scales.size, _ptr(outl), outl.size, q.mean, q.stddev, q.sigma_n,
                                 MEM_HOST, C.byref(w)))
    if out is None:
        out = np.zeros((max(q.rows, 0), max(q.cols, 0)), dtype=np.float32)
    try:
        check(lib().ezq_dequantize_tensor(w, _ptr(out), _mem(out), _stream(stream, out)))
    finally:
        lib().ezq_qweight_free(w)
    return out


def encode_quantized(q: QuantizedWeight) -> bytes:
    """io.hpp:62 encode_quantized: the .ezqt bytes of a host artifact (host
    code, no device needed)."""
    outl = np.ascontiguousarray(q.outliers, dtype=OUTLIER_DTYPE)
    packed = np.ascontiguousarray(q.packed, dtype=np.uint8)
    scales = np.ascontiguousarray(q.scales, dtype=np.float32)
    w = C.POINTER(CQWeight)()
    check(lib().ezq_qweight_wrap(q.rows, q.cols, q.bits, _ptr(packed), packed.size, _ptr(scales),
                                 scales.size, _ptr(outl), outl.size, q.mean, q.stddev, q.sigma_n,
                                 MEM_HOST, C.byref(w)))
    buf = C.POINTER(C.c_uint8)()
    n = C.c_int64(0)
    try:
        check(lib().ezq_encode_quantized(w, C.byref(buf), C.byref(n)))
        return C.string_at(buf, n.value)
    finally:
        lib().ezq_qweight_free(w)
        if buf:
            lib().ezq_free(buf)


def decode_quantized(data: bytes) -> QuantizedWeight:
    """io.hpp:63 decode_quantized; IoError carries the byte offset in .index."""
    arr = np.frombuffer(data, dtype=np.uint8) if len(data) else np.zeros(1, np.uint8)
    q = C.POINTER(CQWeight)()
    check(lib().ezq_decode_quantized(_ptr(arr), len(data), C.byref(q)))
    return _from_c(q.contents, _COwner(q))


def reconstruction_error(a, b, skip: Optional[np.ndarray] = None) -> float:
    a, b = _as_f32(a), _as_f32(b)
    rows, cols = a.shape
    r = c = None
    n = 0
    if skip is not None and len(skip):
        r = np.ascontiguousarray(skip["row"]).astype(np.uint32)
        c = np.ascontiguousarray(skip["col"]).astype(np.uint32)
        n = len(skip)
    out = C.c_double(0)
    check(lib().ezq_reconstruction_error(_ptr(a), _ptr(b), rows, cols, _ptr(r), _ptr(c), n,
                                         _mem(a), None, C.byref(out)))
    return out.value


# ---- channel-scale ----------------------------------------------------------
def _f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


def _mask(m):
    if m is None:
        return None, 0
    m = np.ascontiguousarray(m, dtype=np.uint32)
    return m, m.size


def channel_eval(x, mask, s: float, cfg: Config):
    x = _f32(x)
    m, nm = _mask(mask)
    e, g = C.c_double(0), C.c_double(0)
    c = cfg.to_c()
    check(lib().ezq_channel_eval(_ptr(x), x.size, _ptr(m), nm, s, C.byref(c), C.byref(e), C.byref(g)))
    return e.value, g.value


def optimize_channel(x, mask, cfg: Config, keep_trace: bool = False) -> dict:
    x = _f32(x)
    m, nm = _mask(mask)
    c = cfg.to_c()
    r = COptResult()
    n = max(cfg.steps, 0) + 1
    ts = np.zeros(n, np.int32)
    sc = np.zeros(n, np.float64)
    er = np.zeros(n, np.float64)
    check(lib().ezq_optimize_channel(_ptr(x), x.size, _ptr(m), nm, C.byref(c), int(keep_trace),
                                     C.byref(r), _ptr(ts), _ptr(sc), _ptr(er)))
    k = r.n_trace
    return {"scale": r.scale, "initial_error": r.initial_error, "final_error": r.final_error,
            "best_step": r.best_step, "best_scale": r.best_scale, "best_error": r.best_error,
            "trace_step": ts[:k], "trace_scale": sc[:k], "trace_error": er[:k]}


def brute_force_scale(x, mask, cfg: Config, grid_points: int = 2000):
    x = _f32(x)
    m, nm = _mask(mask)
    c = cfg.to_c()
    s, e = C.c_double(0), C.c_double(0)
    check(lib().ezq_brute_force_scale(_ptr(x), x.size, _ptr(m), nm, C.byref(c), grid_points,
                                      C.byref(s), C.byref(e)))
    return s.value, e.value


def grid_oracle_batch(Ws: Sequence, cfg: Config, grid_points: int = 2000, stream=None):
    """ezq_grid_oracle_batch: the reference's brute-force grid optimum
    (optimize.cpp:186-229) for every column of every tensor, on the device.
    Returns a list of (best_scale, best_error) float64 arrays, one per tensor."""
    Ws = [_as_f32(w) for w in Ws]
    n = len(Ws)
    ptrs = (C.c_void_p * n)(*[_ptr(w) for w in Ws])
    rows = (C.c_int64 * n)(*[w.shape[0] for w in Ws])
    cols = (C.c_int64 * n)(*[w.shape[1] for w in Ws])
    tot = sum(int(w.shape[1]) for w in Ws)
    sc, er = np.zeros(tot, np.float64), np.zeros(tot, np.float64)
    failed = C.c_int(-1)
    c = cfg.to_c()
    check(lib().ezq_grid_oracle_batch(ptrs, rows, cols, n, C.byref(c), grid_points, _mem(Ws[0]),
                                      _stream(stream, Ws[0]), _ptr(sc), _ptr(er), C.byref(failed)))
    out, o = [], 0
    for w in Ws:
        k = int(w.shape[1])
        out.append((sc[o:o + k], er[o:o + k]))
        o += k
    return out


def sigma_sweep_batch(Ws: Sequence, cfg: Config, sigmas: Sequence[float], stream=None):
    """ezq_sigma_sweep_batch: one EASYQUANT batch per sigma_n (the tensor
    stats computed once for device-resident inputs). Returns (n_outliers,
    rtn_error, final_error), each [len(sigmas), len(Ws)]."""
    Ws = [_as_f32(w) for w in Ws]
    n, k = len(Ws), len(sigmas)
    ptrs = (C.c_void_p * n)(*[_ptr(w) for w in Ws])
    rows = (C.c_int64 * n)(*[w.shape[0] for w in Ws])
    cols = (C.c_int64 * n)(*[w.shape[1] for w in Ws])
    sg = np.asarray(sigmas, np.float32)
    no = np.zeros((k, n), np.int64)
    rt, fi = np.zeros((k, n), np.float64), np.zeros((k, n), np.float64)
    failed = C.c_int(-1)
    c = cfg.to_c()
    check(lib().ezq_sigma_sweep_batch(ptrs, rows, cols, n, C.byref(c), _mem(Ws[0]), _stream(stream, Ws[0]),
                                      _ptr(sg), k, _ptr(no), _ptr(rt), _ptr(fi), C.byref(failed)))
    return no, rt, fi


def quantize_channel(x, scale: float, cfg: Config) -> np.ndarray:
    x = _f32(x)
    out = np.zeros(x.size, np.int16)
    c = cfg.to_c()
    check(lib().ezq_quantize_channel(_ptr(x), x.size, scale, C.byref(c), _ptr(out)))
    return out


def initial_scale(x, cfg: Config) -> float:
    x = _f32(x)
    c = cfg.to_c()
    return lib().ezq_initial_scale(_ptr(x), x.size, C.byref(c))


def adam_step(state: dict, scale: float, grad: float, cfg: Config) -> float:
    m, v, t = C.c_double(state["m"]), C.c_double(state["v"]), C.c_int64(state["t"])
    out = C.c_double(0)
    c = cfg.to_c()
    check(lib().ezq_adam_step(C.byref(m), C.byref(v), C.byref(t), scale, grad, C.byref(c), C.byref(out)))
    state.update(m=m.value, v=v.value, t=t.value)
    return out.value


def packed_size(count: int, bits: int) -> int:
    return int(lib().ezq_packed_size(count, bits))


def pack_levels(levels, bits: int) -> np.ndarray:
    lv = np.ascontiguousarray(levels, dtype=np.int16)
    out = np.zeros(packed_size(lv.size, bits), np.uint8)
    check(lib().ezq_pack_levels(_ptr(lv), lv.size, bits, _ptr(out)))
    return out


def unpack_levels(b, count: int, bits: int) -> np.ndarray:
    b = np.ascontiguousarray(b, dtype=np.uint8)
    out = np.zeros(max(count, 0), np.int16)
    check(lib().ezq_unpack_levels(_ptr(b), b.size, count, bits, _ptr(out)))
    return out


def dequantize_channel(levels, scale: float) -> np.ndarray:
    lv = np.ascontiguousarray(levels, dtype=np.int16)
    out = np.zeros(lv.size, np.float32)
    check(lib().ezq_dequantize_channel(_ptr(lv), lv.size, scale, _ptr(out)))
    return out


# ---- dense 3-bit codes (include/ezquant_c.h: ezq_*_dense3) -------------------
def dense3_size(count: int) -> int:
    return int(lib().ezq_dense3_size(count))


def _u8(a):
    if isinstance(a, np.ndarray):
        return np.ascontiguousarray(a, dtype=np.uint8)
    import torch
    if a.dtype != torch.uint8 or not a.is_contiguous():
        raise ValueError("dense3: expected a contiguous uint8 tensor")
    return a


def pack_dense3(levels, stream=None):
    """The k = 3 payload (one offset byte per level; numpy or torch uint8, all
    host or all device) -> dense 3-bit stream in the same memory."""
    lv = _u8(levels)
    n = int(lv.size if isinstance(lv, np.ndarray) else lv.numel())
    if isinstance(lv, np.ndarray):
        out = np.zeros(dense3_size(n), np.uint8)
    else:
        import torch
        out = torch.empty(dense3_size(n), dtype=torch.uint8, device=lv.device)
    check(lib().ezq_pack_dense3(_ptr(lv), n, _ptr(out), _mem(lv), _stream(stream, lv)))
    return out


def unpack_dense3(dense, count: int, stream=None):
    """Dense 3-bit stream -> one offset byte per level (same memory kind)."""
    d = _u8(dense)
    if isinstance(d, np.ndarray):
        out = np.zeros(max(count, 0), np.uint8)
    else:
        import torch
        out = torch.empty(max(count, 0), dtype=torch.uint8, device=d.device)
    check(lib().ezq_unpack_dense3(_ptr(d), count, _ptr(out), _mem(d), _stream(stream, d)))
    return out


def dequantize_dense3(q: "QuantizedWeight", dense, out=None, stream=None) -> np.ndarray:
    """dequantize_tensor of a host 3-bit artifact whose codes are the dense
    stream `dense` (numpy uint8)."""
    outl = np.ascontiguousarray(q.outliers, dtype=OUTLIER_DTYPE)
    scales = np.ascontiguousarray(q.scales, dtype=np.float32)
    d = np.ascontiguousarray(dense, dtype=np.uint8)
    w = C.POINTER(CQWeight)()
    check(lib().ezq_qweight_wrap(q.rows, q.cols, q.bits, None, 0, _ptr(scales), scales.size, _ptr(outl),
                                 outl.size, q.mean, q.stddev, q.sigma_n, MEM_HOST, C.byref(w)))
    if out is None:
        out = np.zeros((max(q.rows, 0), max(q.cols, 0)), dtype=np.float32)
    try:
        check(lib().ezq_dequantize_dense3(w, _ptr(d), _ptr(out), _mem(out), _stream(stream, out)))
    finally:
        lib().ezq_qweight_free(w)
    return out


class GemvPlanDense3(GemvPlan):
    """GemvPlan of a device-resident 3-bit DeviceBatch entry whose codes are
    given as a dense 3-bit stream on the device (torch uint8)."""

    def __init__(self, batch: "DeviceBatch", i: int, dense, stream=None, outlier_dtype: str = "float32"):
        self._keep = (batch, dense)
        self.rows, self.cols = batch[i].rows, batch[i].cols
        self.p = C.c_void_p()
        check(lib().ezq_gemv_prepare_dense3(batch.ptrs[i], _ptr(_u8(dense)), self.OUTLIER_DTYPES[outlier_dtype],
                                            _stream(stream, dense), C.byref(self.p)))
        self.stream = stream

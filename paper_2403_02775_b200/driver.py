"""Whole-model driver across the GPUs of one node (one process per GPU).

Mirrors quantize_model (model.cpp:123-212): tensors are independent units
(one OpenMP task per tensor there, one LPT bin per GPU here), 1-D /
degenerate tensors pass through unquantized (model.cpp:147,174-177), a bad
tensor fails alone (model.cpp:160-186), and the result is independent of the
worker (here: rank) count. No collective touches the data path.

Two forms:
- quantize_model_sharded(manifest, out_dir, ...): the on-disk driver. Every
  rank runs the C++ drop-in driver (csrc/model.cpp quantize_model_shard) on
  its LPT share -- reading, quantizing in device batches and writing the
  .ezqt files itself -- then rank 0 merges the per-rank records into
  quantized_manifest.json. The directory is byte-identical to a
  single-process quantize_model (and so to the reference's). torch.distributed
  is used for one barrier only.
- quantize_sharded(tensors, ...): in-memory tensors (numpy or CUDA), this
  rank's LPT share quantized with ezq_quantize_batch; optionally gathered on
  rank 0 (small models -- large ones use the on-disk form).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np


def lpt_partition(sizes: Sequence[int], world: int) -> List[List[int]]:
    """Longest-processing-time-first bins (work ~ rows*cols); deterministic
    (ties broken by index, then by rank), each bin sorted by tensor index.
    Same rule as the C++ lpt_shards (csrc/model.cpp)."""
    bins: List[List[int]] = [[] for _ in range(world)]
    load = [0] * world
    for i in sorted(range(len(sizes)), key=lambda k: (-sizes[k], k)):
        r = min(range(world), key=lambda b: (load[b], b))
        bins[r].append(i)
        load[r] += sizes[i]
    return [sorted(b) for b in bins]


# ---- on-disk driver (C++ drop-in through include/ezquant_model_c.h) -----------
_mlib = None


def model_lib() -> C.CDLL:
    """libezquant.so (the C++ drop-in) and its model-driver C-ABI."""
    global _mlib
    if _mlib is None:
        from . import native
        native.lib()  # loads libezq_b200.so first (dependency)
        L = C.CDLL(os.path.join(os.path.dirname(native.LIB_PATH), "libezquant.so"))
        P, I32, I64 = C.c_char_p, C.c_int, C.c_int64
        cfgp = C.POINTER(native.CConfig)
        L.ezqm_quantize_model.argtypes = [P, P, cfgp, I32, I32, C.POINTER(I32), C.c_char_p, C.c_size_t]
        L.ezqm_quantize_model_shard.argtypes = [P, P, cfgp, I32, I32, I32, I32, C.POINTER(I32), C.c_char_p,
                                                C.c_size_t]
        L.ezqm_merge_model_shards.argtypes = [P, P, cfgp, I32, I32, C.POINTER(I32), C.c_char_p, C.c_size_t]
        L.ezqm_lpt_shard.argtypes = [P, I32, I32, C.POINTER(I64), I64]
        L.ezqm_lpt_shard.restype = I64
        _mlib = L
    return _mlib


def _call(fn, *args) -> int:
    from . import native
    buf = C.create_string_buffer(4096)
    fails = C.c_int(0)
    code = fn(*args, C.byref(fails), buf, len(buf))
    if code != 0:
        raise native.EzqError(code, buf.value.decode(errors="replace"), -1)
    return fails.value


def quantize_model(manifest: str, out_dir: str, cfg, mode: str = "easyquant", workers: int = 4) -> int:
    """Single-process quantize_model (model.hpp:63); returns the failure count."""
    from . import native
    c = cfg.to_c()
    return _call(model_lib().ezqm_quantize_model, manifest.encode(), out_dir.encode(), C.byref(c),
                 native.MODES[mode], workers)


def lpt_shard(manifest: str, rank: int, world: int) -> List[int]:
    """This rank's manifest indices (the C++ lpt_shards bin)."""
    idx = (C.c_int64 * 1)()
    n = model_lib().ezqm_lpt_shard(manifest.encode(), rank, world, idx, 0)
    if n < 0:
        raise ValueError(f"cannot partition {manifest}")
    idx = (C.c_int64 * max(n, 1))()
    model_lib().ezqm_lpt_shard(manifest.encode(), rank, world, idx, n)
    return [int(v) for v in idx[:n]]


def quantize_model_shard(manifest: str, out_dir: str, cfg, mode: str, rank: int, world: int,
                         workers: int = 4) -> int:
    from . import native
    c = cfg.to_c()
    return _call(model_lib().ezqm_quantize_model_shard, manifest.encode(), out_dir.encode(), C.byref(c),
                 native.MODES[mode], workers, rank, world)


def merge_model_shards(manifest: str, out_dir: str, cfg, mode: str, world: int) -> int:
    from . import native
    c = cfg.to_c()
    return _call(model_lib().ezqm_merge_model_shards, manifest.encode(), out_dir.encode(), C.byref(c),
                 native.MODES[mode], world)


def quantize_model_sharded(manifest: str, out_dir: str, cfg, mode: str = "easyquant", rank: int = 0,
                           world: int = 1, workers: int = 4, group=None) -> int:
    """quantize_model over `world` processes (one per GPU): this rank's LPT
    share is quantized and written by the C++ driver; after a barrier rank 0
    writes the merged manifest. Returns the failure count (rank 0: all
    tensors; other ranks: their own). A rank whose shard raised still reaches
    the barrier and re-raises after it; rank 0's merge then fails on the
    missing shard record -- no rank waits forever."""
    err = None
    try:
        fails = quantize_model_shard(manifest, out_dir, cfg, mode, rank, world, workers)
    except Exception as e:  # noqa: BLE001 -- re-raised after the barrier
        err, fails = e, 0
    if world > 1:
        import torch.distributed as dist
        dist.barrier(group=group)
    if err is not None:
        raise err
    if rank != 0:
        return fails
    return merge_model_shards(manifest, out_dir, cfg, mode, world)


# ---- in-memory driver --------------------------------------------------------
def _default_quantize(mats, cfg, mode):
    from . import native
    return native.quantize_batch(mats, cfg, mode)


def _finite(w) -> bool:
    if isinstance(w, np.ndarray):
        return bool(np.isfinite(w).all())
    import torch
    return bool(torch.isfinite(w).all())


def quantize_sharded(tensors: Sequence[Tuple[str, object]], cfg, mode: str = "easyquant",
                     rank: int = 0, world: int = 1, group=None,
                     quantize_fn: Optional[Callable] = None, gather: bool = True) -> Optional[Dict[str, object]]:
    """Quantizes this rank's LPT share of `tensors` ((name, 2-D array) pairs,
    numpy or CUDA tensors). Returns {name: artifact | ("passthrough", array) |
    ("failed", message)}: on rank 0 for every tensor (gathered as picklable
    host artifacts) when `gather`, else this rank's share on every rank.

    Per-tensor semantics follow model.cpp:160-186: a batch that raises is
    re-run tensor by tensor, so one bad tensor fails alone and every rank
    still reaches the gather; degenerate matrices (rows == 1 or cols == 1)
    pass through after the finiteness check DenseMatrix::validate applies
    (types.cpp:9-21)."""
    quantize_fn = quantize_fn or _default_quantize
    sizes = [int(np.prod(w.shape)) for _, w in tensors]
    mine = lpt_partition(sizes, world)[rank]
    out: Dict[str, object] = {}
    todo = []
    for i in mine:
        name, w = tensors[i]
        if min(w.shape) <= 1:
            out[name] = ("passthrough", w) if _finite(w) else ("failed", f"{name}: non-finite value")
        else:
            todo.append(i)
    if todo:
        try:
            arts = quantize_fn([tensors[i][1] for i in todo], cfg, mode)
            out.update({tensors[i][0]: a for i, a in zip(todo, arts)})
        except Exception:  # noqa: BLE001 -- attribute the failure tensor by tensor
            for i in todo:
                try:
                    out[tensors[i][0]] = quantize_fn([tensors[i][1]], cfg, mode)[0]
                except Exception as e:  # noqa: BLE001
                    out[tensors[i][0]] = ("failed", str(e))
    if world == 1 or not gather:
        return out
    import torch.distributed as dist
    host = {}
    for k, v in out.items():  # device tensors / library views -> plain host objects
        if isinstance(v, tuple) and v[0] == "passthrough" and not isinstance(v[1], np.ndarray):
            v = ("passthrough", v[1].cpu().numpy())
        host[k] = v
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(host, gathered, dst=0, group=group)
    if rank != 0:
        return None
    merged: Dict[str, object] = {}
    for part in gathered:
        merged.update(part)
    return {name: merged[name] for name, _ in tensors}

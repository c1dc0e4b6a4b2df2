"""Whole-model driver: shards independent weight matrices across the GPUs of
one node (one process per GPU), quantizes each rank's share with grouped
launches (ezq_quantize_batch), and gathers the artifacts on rank 0.

Mirrors quantize_model (model.cpp:123-212): tensors are independent units
(one task per tensor there, one LPT bin per GPU here), 1-D / degenerate
tensors pass through unquantized (model.cpp:147,174-177), and the result is
independent of the worker (here: rank) count. No collective touches the data
path -- torch.distributed is only used to gather the (small) artifacts.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np


def lpt_partition(sizes: Sequence[int], world: int) -> List[List[int]]:
    """Longest-processing-time-first bins (work ~ rows*cols); deterministic
    (ties broken by index), each bin sorted by tensor index."""
    bins: List[List[int]] = [[] for _ in range(world)]
    load = [0] * world
    for i in sorted(range(len(sizes)), key=lambda k: (-sizes[k], k)):
        r = min(range(world), key=lambda b: (load[b], b))
        bins[r].append(i)
        load[r] += sizes[i]
    return [sorted(b) for b in bins]


def _default_quantize(mats, cfg, mode):
    from . import native
    return native.quantize_batch(mats, cfg, mode)


def quantize_sharded(tensors: Sequence[Tuple[str, object]], cfg, mode: str = "easyquant",
                     rank: int = 0, world: int = 1, group=None,
                     quantize_fn: Optional[Callable] = None) -> Optional[Dict[str, object]]:
    """Quantizes this rank's LPT share of `tensors` ((name, 2-D array) pairs,
    numpy or CUDA tensors) and gathers {name: artifact} on rank 0 (None on
    other ranks). Degenerate matrices (rows == 1 or cols == 1) pass through
    as-is, like the reference model driver."""
    quantize_fn = quantize_fn or _default_quantize
    sizes = [int(np.prod(w.shape)) for _, w in tensors]
    mine = lpt_partition(sizes, world)[rank]
    todo = [i for i in mine if min(tensors[i][1].shape) > 1]
    passthrough = {tensors[i][0]: ("passthrough", tensors[i][1]) for i in mine
                   if min(tensors[i][1].shape) <= 1}
    out = dict(passthrough)
    if todo:
        arts = quantize_fn([tensors[i][1] for i in todo], cfg, mode)
        out.update({tensors[i][0]: a for i, a in zip(todo, arts)})
    if world == 1:
        return out
    import torch.distributed as dist
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(out, gathered, dst=0, group=group)
    if rank != 0:
        return None
    merged: Dict[str, object] = {}
    for part in gathered:
        merged.update(part)
    return {name: merged[name] for name, _ in tensors}

"""CPU, world_size 2 over gloo: the multi-GPU model driver's sharding and
artifact gather. The per-rank quantizer is injected (the C restatement,
test infrastructure) because this container has no GPU; on the B200 the
same driver calls ezq_quantize_batch."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_02775_b200.driver import lpt_partition, quantize_sharded
from paper_2403_02775_b200.native import Config


def test_lpt_partition_balanced_and_complete():
    sizes = [4 * 2048 * 2048] * 4 * 24 + [2048 * 8192] * 48   # OPT-1.3B set
    for world in (1, 2, 4, 8):
        bins = lpt_partition(sizes, world)
        assert sorted(i for b in bins for i in b) == list(range(len(sizes)))
        loads = [sum(sizes[i] for i in b) for b in bins]
        assert max(loads) - min(loads) <= max(sizes)
    assert lpt_partition([5, 3, 3, 1], 2) == [[0, 3], [1, 2]]


def _oracle_quantize(mats, cfg, mode):
    from oracle import pyoracle
    return [pyoracle.quantize(np.asarray(W), cfg, mode, threads=1) for W in mats]


def _model():
    from oracle import pyoracle
    names = ["blocks.%d.%s" % (l, p) for l in range(3) for p in ("wq", "w1", "w2")]
    shapes = [(48, 48), (48, 96), (96, 48)] * 3
    mats = [pyoracle.gaussian(r, c, 10 + i, 0.05) for i, (r, c) in enumerate(shapes)]
    mats.append(pyoracle.gaussian(1, 64, 99, 0.05))   # 1-D bias: passthrough
    names.append("blocks.0.bias")
    return list(zip(names, mats))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = quantize_sharded(_model(), Config(steps=20), "easyquant", rank, world,
                           quantize_fn=_oracle_quantize)
    if rank == 0:
        q.put({k: (v[0] if isinstance(v, tuple) else (v["packed"].tobytes(), v["scales"].tobytes(),
                                                        v["final_error"]))
               for k, v in res.items()})
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    single = quantize_sharded(_model(), Config(steps=20), "easyquant", 0, 1,
                              quantize_fn=_oracle_quantize)
    assert list(got) == [n for n, _ in _model()]
    for name, art in single.items():
        if isinstance(art, tuple):
            assert got[name] == "passthrough"
        else:
            assert got[name] == (art["packed"].tobytes(), art["scales"].tobytes(), art["final_error"])

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


def _raising_quantize(mats, cfg, mode):
    """The oracle quantizer; raises on a non-finite tensor like ezq_quantize_batch."""
    from oracle import pyoracle
    out = []
    for W in mats:
        if not np.isfinite(np.asarray(W)).all():
            raise ValueError("non-finite element")
        out.append(pyoracle.quantize(np.asarray(W), cfg, mode, threads=1))
    return out


def _fail_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model = _model()
    W = model[1][1].copy()
    W[2, 3] = np.nan
    model[1] = (model[1][0], W)                         # one bad matrix
    b = model[-1][1].copy()
    b[0, 1] = np.inf
    model[-1] = (model[-1][0], b)                       # one bad vector
    res = quantize_sharded(model, Config(steps=10), "easyquant", rank, world, quantize_fn=_raising_quantize)
    if rank == 0:
        q.put({k: (v[0] if isinstance(v, tuple) else "ok") for k, v in res.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_failure_is_per_tensor():
    """model.cpp:160-186: a tensor that fails (non-finite) fails alone -- the
    rank re-runs its batch tensor by tensor and still reaches the gather."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fail_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    names = [n for n, _ in _model()]
    assert got[names[1]] == "failed" and got[names[-1]] == "failed"
    assert all(got[n] == "ok" for n in names[:-1] if n != names[1])


def test_lpt_cpp_matches_python(N, tmp_path):
    """The C++ driver's LPT bins (csrc/model.cpp lpt_shards) equal lpt_partition."""
    import json
    from paper_2403_02775_b200.driver import lpt_shard
    shapes = ([(2048, 2048)] * 4 + [(2048, 8192), (8192, 2048), (1, 2048)]) * 5 + [(3, 3), (5, 1)]
    man = {"version": 1, "tensors": [{"name": f"t{i}", "rows": r, "cols": c, "dtype": "f32", "file": f"t{i}.raw"}
                                     for i, (r, c) in enumerate(shapes)]}
    path = tmp_path / "manifest.json"
    path.write_text(json.dumps(man))
    for world in (1, 2, 3, 8):
        bins = lpt_partition([r * c for r, c in shapes], world)
        assert [lpt_shard(str(path), r, world) for r in range(world)] == bins


def _disk_model(d):
    import json
    os.makedirs(d, exist_ok=True)
    from oracle import pyoracle
    tensors = []
    for i, (r, c) in enumerate([(64, 32), (1, 32), (48, 96), (96, 1), (32, 32), (1, 7)]):
        W = pyoracle.gaussian(r, c, 50 + i, 0.05)
        W.astype("<f4").tofile(os.path.join(d, f"t{i}.raw"))
        tensors.append({"name": f"layer.{i}", "rows": r, "cols": c, "dtype": "f32", "file": f"t{i}.raw"})
    tensors.append({"name": "missing", "rows": 4, "cols": 4, "dtype": "f32", "file": "nope.raw"})
    with open(os.path.join(d, "manifest.json"), "w") as f:
        json.dump({"version": 1, "tensors": tensors}, f)
    return os.path.join(d, "manifest.json")


def _disk_worker(rank, world, port, man, out, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2403_02775_b200.driver import quantize_model_sharded
    fails = quantize_model_sharded(man, out, Config(steps=10), "easyquant", rank, world, workers=2)
    if rank == 0:
        q.put(fails)
    dist.destroy_process_group()


def test_model_sharded_equals_single_process(N, tmp_path):
    """The on-disk multi-process driver (world 2 over gloo) writes the same
    directory, byte for byte, as the single-process quantize_model. Here (no
    GPU) every matrix is a per-tensor NO_DEVICE failure and the vectors pass
    through; the B200 test (test_model_driver.py) covers the quantized files."""
    from paper_2403_02775_b200.driver import quantize_model
    man = _disk_model(str(tmp_path / "in"))
    single, sharded = str(tmp_path / "single"), str(tmp_path / "sharded")
    n_single = quantize_model(man, single, Config(steps=10), "easyquant", workers=2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_disk_worker, args=(r, 2, port, man, sharded, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got == n_single
    a, b = sorted(os.listdir(single)), sorted(os.listdir(sharded))
    assert a == b and "quantized_manifest.json" in a
    for name in a:
        with open(os.path.join(single, name), "rb") as f1, open(os.path.join(sharded, name), "rb") as f2:
            assert f1.read() == f2.read(), name

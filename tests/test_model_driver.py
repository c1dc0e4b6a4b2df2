"""The whole-model driver (model.hpp quantize_model / dequantize_model, SURVEY
§8f next #1) through the C++ drop-in: the output directory -- every .ezqt,
every pass-through .bin and quantized_manifest.json / manifest.json -- must
be byte-identical to the compiled reference's on the same manifest,
including per-tensor failures (missing file, short file, non-finite values)
and for any worker count."""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_2403_02775_b200", "_lib")


def _tool(tmp_path):
    exe = str(tmp_path / "model_tool")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "model_tool.cpp"), "-L" + LIB, "-lezquant",
                    "-lezq_b200", "-Wl,-rpath," + LIB, "-o", exe], check=True)
    return exe


def _model(d, O):
    """A small model: matrices of several shapes (roles/layers), a bias
    vector, a missing file, a short file and a non-finite tensor."""
    os.makedirs(d, exist_ok=True)
    tensors = []

    def add(name, rows, cols, seed, role=None, layer=None, data=None, write=True):
        fname = name.replace("/", "_") + ".raw"
        if write:
            W = data if data is not None else O.gaussian(rows, cols, seed, 0.02)
            if data is None and rows > 1 and cols > 1:
                O.plant_outliers(W, max(1, rows * cols // 500), 0.2, 1.0, seed + 1)
            W.astype("<f4").tofile(os.path.join(d, fname))
        e = {"name": name, "rows": rows, "cols": cols, "dtype": "f32", "file": fname}
        if role:
            e["role"] = role
        if layer is not None:
            e["layer"] = layer
        tensors.append(e)

    add("blocks.0.attn.wq", 256, 128, 1, "attention", 0)
    add("blocks.0.attn.bias", 1, 128, 2, "attention", 0)
    add("blocks.0.mlp.w1", 128, 512, 3, "mlp", 0)
    add("blocks.0.mlp/w2:odd name", 513, 77, 4, "mlp", 0)
    add("blocks.1.norm", 96, 1, 5, "norm", 1)
    add("embed", 300, 64, 6)
    add("missing", 16, 16, 7, write=False)
    short = np.ones((4, 4), np.float32)
    add("short", 8, 4, 8, data=short)
    bad = O.gaussian(32, 24, 9, 0.02)
    bad[3, 5] = np.inf
    add("nonfinite", 32, 24, 9, data=bad)
    with open(os.path.join(d, "manifest.json"), "w") as f:
        json.dump({"version": 1, "tensors": tensors}, f, indent=2)
    return os.path.join(d, "manifest.json")


def _tree(d):
    out = {}
    for name in sorted(os.listdir(d)):
        with open(os.path.join(d, name), "rb") as f:
            out[name] = f.read()
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("mode,bits,workers", [("easyquant", 4, 1), ("easyquant", 3, 4),
                                               ("rtn", 4, 2), ("outliers-only", 4, 3)])
def test_quantize_model_byte_identical_to_reference(gpu, O, tmp_path, mode, bits, workers):
    from oracle import refimpl as R
    if not R.available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    from paper_2403_02775_b200.native import Config
    man = _model(str(tmp_path / "in"), O)
    cfg = Config(bits=bits, steps=40)
    ref_out, our_out = str(tmp_path / "ref"), str(tmp_path / "ours")
    ref_fail = R.quantize_model(man, ref_out, cfg, mode, workers=workers)
    exe = _tool(tmp_path)
    r = subprocess.run([exe, "quantize", man, our_out, str(bits), str(cfg.sigma_n), mode, "40",
                        str(workers)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert f"failures {ref_fail}" in r.stdout, r.stdout
    assert ref_fail == 3  # missing, short, non-finite
    ref_tree, our_tree = _tree(ref_out), _tree(our_out)
    assert sorted(ref_tree) == sorted(our_tree)
    for name in ref_tree:
        assert our_tree[name] == ref_tree[name], name

    # and back: dequantize_model output is byte-identical too
    ref_dq, our_dq = str(tmp_path / "ref_dq"), str(tmp_path / "ours_dq")
    assert R.dequantize_model(ref_out, ref_dq, workers=workers) == 0
    r = subprocess.run([exe, "dequantize", our_out, our_dq, str(workers)], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "failures 0" in r.stdout, r.stdout + r.stderr
    a, b = _tree(ref_dq), _tree(our_dq)
    assert sorted(a) == sorted(b)
    for name in a:
        assert a[name] == b[name], name


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_quantize_model_sharded_byte_identical(gpu, O, tmp_path, world):
    """The multi-GPU on-disk driver (driver.quantize_model_sharded: every rank
    quantizes its LPT share with the C++ driver, rank 0 merges the manifest):
    the directory equals the compiled reference's quantize_model byte for
    byte. The ranks run one after another in this process (one GPU here; the
    shards share no state -- the gloo test covers the multi-process barrier)."""
    from oracle import refimpl as R
    if not R.available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    from paper_2403_02775_b200 import driver
    from paper_2403_02775_b200.native import Config
    man = _model(str(tmp_path / "in"), O)
    cfg = Config(bits=4, steps=40)
    ref_out, our_out = str(tmp_path / "ref"), str(tmp_path / "ours")
    ref_fail = R.quantize_model(man, ref_out, cfg, "easyquant", workers=2)
    for r in range(world):
        driver.quantize_model_shard(man, our_out, cfg, "easyquant", r, world, workers=2)
    assert driver.merge_model_shards(man, our_out, cfg, "easyquant", world) == ref_fail
    ref_tree, our_tree = _tree(ref_out), _tree(our_out)
    assert sorted(ref_tree) == sorted(our_tree)
    for name in ref_tree:
        assert our_tree[name] == ref_tree[name], name


@pytest.mark.gpu
def test_sigma_sweep_matches_reference(gpu, O, tmp_path):
    """report.hpp sigma_sweep: per-sigma outlier counts/fractions and the
    manifest-order error sums are bit-identical to the reference's (compared
    as sweep_to_json text)."""
    from oracle import refimpl as R
    if not R.available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    from paper_2403_02775_b200.native import Config
    d = str(tmp_path / "in")
    man = _model(d, O)
    # the sweep requires every 2-D tensor to load: keep the good ones
    with open(man) as f:
        m = json.load(f)
    m["tensors"] = [t for t in m["tensors"] if t["name"] not in ("missing", "short", "nonfinite")]
    with open(man, "w") as f:
        json.dump(m, f)
    sigmas = [1.5, 2.0, 2.5758, 3.0, 4.0]
    ref = R.sigma_sweep(man, Config(bits=4, steps=30), sigmas, workers=4)
    exe = _tool(tmp_path)
    r = subprocess.run([exe, "sweep", man, "4", "30", "3"] + [repr(s) for s in sigmas],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout == ref


def test_model_tool_compiles(N, tmp_path):
    """CPU: a reference-style whole-model caller builds against the drop-in."""
    _tool(tmp_path)

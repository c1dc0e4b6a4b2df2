"""Dense 3-bit codes (include/ezquant_c.h ezq_*_dense3).

CPU: the numpy restatement of the layout (oracle/pyoracle.py) against a
hand-computed vector, round trips and sizes. GPU: the device codec against the
restatement (bit-exact), pack/unpack/dequantize round trips on real 3-bit
artifacts (dequantize from the dense stream is bit-identical to
ezq_dequantize_tensor on the reference's byte-per-level codes), the span check,
ragged counts, and a GEMV plan built from the dense stream giving the same y as
the plan built from the byte codes.
"""
import numpy as np
import pytest

from oracle import pyoracle as O


def test_dense3_layout_known_answer():
    # offsets 0..7: bits 3e..3e+2 of 0b111_110_101_100_011_010_001_000 = 0xFAC688
    s = O.dense3_pack(np.arange(8, dtype=np.uint8))
    assert s.tolist() == [0x88, 0xC6, 0xFA]
    assert O.dense3_unpack(s, 8).tolist() == list(range(8))
    # a ragged tail: 3 offsets use one 3-byte group with zero tail bits
    s = O.dense3_pack(np.array([7, 0, 5], np.uint8))
    assert s.tolist() == [0x47, 0x01, 0x00]  # 7 | 5 << 6


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 31, 32, 33, 1000, 4099])
def test_dense3_oracle_roundtrip(n):
    rng = np.random.default_rng(n)
    o = rng.integers(0, 8, n, dtype=np.uint8)
    s = O.dense3_pack(o)
    assert s.size == O.dense3_size(n) == (0 if n == 0 else 3 * ((n + 7) // 8))
    assert np.array_equal(O.dense3_unpack(s, n), o)


def test_dense3_oracle_rejects_wide_offsets():
    with pytest.raises(ValueError):
        O.dense3_pack(np.array([0, 8], np.uint8))


def test_dense3_size_matches_oracle(N):
    for n in (0, 1, 8, 9, 123457):
        assert N.dense3_size(n) == O.dense3_size(n)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 7, 8, 31, 32, 33, 4095, 100003, 1 << 22])
def test_dense3_codec_gpu(gpu, n):
    import torch
    from paper_2403_02775_b200 import native as N
    rng = np.random.default_rng(n)
    o = rng.integers(0, 8, n, dtype=np.uint8)
    ref = O.dense3_pack(o)
    s = N.pack_dense3(o)  # host buffers
    assert np.array_equal(s, ref)
    assert np.array_equal(N.unpack_dense3(s, n), o)
    od = torch.from_numpy(o).cuda()  # device buffers
    sd = N.pack_dense3(od)
    assert np.array_equal(sd.cpu().numpy(), ref)
    assert np.array_equal(N.unpack_dense3(sd, n).cpu().numpy(), o)


@pytest.mark.gpu
def test_dense3_unaligned_buffers_gpu(gpu):
    import torch
    from paper_2403_02775_b200 import native as N
    n = 5000
    o = np.random.default_rng(5).integers(0, 8, n, dtype=np.uint8)
    base = torch.zeros(n + 16, dtype=torch.uint8, device="cuda")
    od = base[3:3 + n]
    od.copy_(torch.from_numpy(o).cuda())
    sbase = torch.zeros(O.dense3_size(n) + 8, dtype=torch.uint8, device="cuda")
    sd = sbase[1:1 + O.dense3_size(n)]
    from paper_2403_02775_b200.native import lib, check, MEM_DEVICE
    check(lib().ezq_pack_dense3(od.data_ptr(), n, sd.data_ptr(), MEM_DEVICE, None))
    torch.cuda.synchronize()
    assert np.array_equal(sd.cpu().numpy(), O.dense3_pack(o))
    ub = torch.zeros(n + 8, dtype=torch.uint8, device="cuda")[5:5 + n]
    check(lib().ezq_unpack_dense3(sd.data_ptr(), n, ub.data_ptr(), MEM_DEVICE, None))
    torch.cuda.synchronize()
    assert np.array_equal(ub.cpu().numpy(), o)


@pytest.mark.gpu
def test_dense3_span_check_gpu(gpu):
    from paper_2403_02775_b200 import native as N
    o = np.zeros(100, np.uint8)
    o[37] = 8
    o[60] = 200
    with pytest.raises(N.InvalidArgument) as ei:
        N.pack_dense3(o)
    assert "exceeds level span 7" in str(ei.value)
    assert ei.value.index == 37  # the first offending element


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols", [(64, 40), (1000, 333), (4096, 4096)])
def test_dense3_dequantize_matches_bytes_gpu(gpu, rows, cols):
    from paper_2403_02775_b200 import native as N
    from paper_2403_02775_b200.native import Config
    W = O.gaussian(rows, cols, rows + cols, 0.02)
    O.plant_outliers(W, max(1, rows * cols // 200), 0.2, 1.0, 11)
    q = N.quantize_tensor(W, Config(bits=3, steps=20))
    dense = N.pack_dense3(q.packed)
    assert dense.size == O.dense3_size(rows * cols)
    assert np.array_equal(dense, O.dense3_pack(q.packed))
    ref = N.dequantize(q)
    got = N.dequantize_dense3(q, dense)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


@pytest.mark.gpu
def test_dense3_device_batch_and_gemv_gpu(gpu):
    import torch
    from paper_2403_02775_b200 import native as N
    from paper_2403_02775_b200.native import Config
    rows, cols = 4096, 1100
    g = torch.Generator(device="cuda").manual_seed(7)
    Wd = torch.randn(rows, cols, generator=g, device="cuda") * 0.02
    b = N.quantize_batch([Wd], Config(bits=3, sigma_n=2.5758, steps=20), out_mem=N.MEM_DEVICE)
    codes = torch.from_numpy(b.to_host(0).packed.copy()).cuda()  # the byte-per-level k = 3 payload
    dense = N.pack_dense3(codes)
    assert np.array_equal(N.unpack_dense3(dense, rows * cols).cpu().numpy(), codes.cpu().numpy())
    out_b = torch.empty(rows, cols, device="cuda")
    out_d = torch.empty(rows, cols, device="cuda")
    b.dequantize_into(0, out_b)
    b.dequantize_dense3_into(0, dense, out_d)
    torch.cuda.synchronize()
    assert torch.equal(out_b.view(torch.int32), out_d.view(torch.int32))
    x = torch.randn(3, rows, generator=g, device="cuda").to(torch.bfloat16)
    p1 = N.GemvPlan(b, 0)
    p2 = N.GemvPlanDense3(b, 0, dense)
    y1, y2 = p1(x), p2(x)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)  # the same plan: bit-identical outputs
    p1.close()
    p2.close()
    b.close()


def test_dense3_wrapper_rejects_non_u8_tensors(N):
    import torch
    with pytest.raises(ValueError):
        N.pack_dense3(torch.zeros(16, dtype=torch.int16))
    with pytest.raises(ValueError):
        N.unpack_dense3(torch.zeros(6, dtype=torch.uint8)[::2], 4)


@pytest.mark.gpu
def test_dense3_null_buffers_gpu(gpu):
    from paper_2403_02775_b200.native import lib, MEM_DEVICE, MEM_HOST, INVALID_ARGUMENT
    assert lib().ezq_pack_dense3(None, 10, None, MEM_HOST, None) == INVALID_ARGUMENT
    assert lib().ezq_unpack_dense3(None, 10, None, MEM_DEVICE, None) == INVALID_ARGUMENT
    assert lib().ezq_pack_dense3(None, 0, None, MEM_HOST, None) == 0  # empty: no-op

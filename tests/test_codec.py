"""CPU: the .ezqt container codec (ezq_encode_quantized / ezq_decode_quantized,
host code) against the reference's test_io.cpp cases and golden fixture, and
-- where oracle/_ref exists -- byte-for-byte against the compiled reference
encoder/decoder on seeded artifacts and corrupted buffers (categories and
byte offsets)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN

OUTLIER = [("row", "<u4"), ("col", "<u4"), ("value", "<f4")]


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "golden_1x2.ezqt"), "rb") as f:
        return f.read()


@pytest.fixture(scope="module")
def R():
    from oracle import refimpl
    if not refimpl.available():
        pytest.skip("compiled reference (oracle/_ref) not built here")
    return refimpl


def _artifact(N, O, rows, cols, bits, seed, n_out=3):
    """An artifact from the oracle's quantizer (C restatement, CPU)."""
    W = O.gaussian(rows, cols, seed, 0.05)
    O.plant_outliers(W, n_out, 2.0, 4.0, seed + 1)
    cfg = N.Config(bits=bits, steps=10)
    r = O.quantize(W, cfg)
    return N.QuantizedWeight(rows, cols, bits, r["packed"], r["scales"], r["outliers"],
                             r["mean"], r["stddev"], cfg.sigma_n)


def test_golden_decodes_to_documented_contents(N, golden):
    """test_io.cpp:137-151"""
    q = N.decode_quantized(golden)
    assert (q.rows, q.cols, q.bits) == (1, 2, 4)
    assert q.sigma_n == 1.0 and q.mean == 50.5 and q.stddev == 49.5
    assert q.scales.tolist() == [1.0, 1.0]
    assert [tuple(e) for e in q.outliers.tolist()] == [(0, 0, 1.0), (0, 1, 100.0)]
    assert q.packed.tolist() == [0x77]
    assert q.rtn_error is None and q.final_error is None  # provenance is not in the file


def test_golden_reencodes_bit_exactly(N, golden):
    assert N.encode_quantized(N.decode_quantized(golden)) == golden


@pytest.mark.parametrize("bits", [2, 3, 4, 5, 8])
def test_round_trip_every_field(N, O, bits):
    """test_io.cpp:92-100"""
    q = _artifact(N, O, 17, 9, bits, 7 + bits)
    b = N.encode_quantized(q)
    back = N.decode_quantized(b)
    assert (back.rows, back.cols, back.bits) == (q.rows, q.cols, q.bits)
    assert np.array_equal(back.packed, q.packed)
    assert np.array_equal(back.scales.view(np.uint32), q.scales.view(np.uint32))
    assert np.array_equal(back.outliers, q.outliers)
    assert (back.mean, back.stddev, back.sigma_n) == (q.mean, q.stddev, np.float32(q.sigma_n))
    assert len(b) == 48 + 4 * q.cols + 8 + 12 * len(q.outliers) + q.packed.size


def _expect_io(N, data, code, offset=None, text=None):
    with pytest.raises(N.IoError) as ei:
        N.decode_quantized(bytes(data))
    assert ei.value.code == code
    if offset is not None:
        assert ei.value.index == offset
    if text is not None:
        assert text in ei.value.msg
    return ei.value


def test_decoder_rejects_corrupted_buffers(N, golden):
    """test_io.cpp:153-234 (category and offset of every corruption)."""
    g = bytearray(golden)
    FMT, VER = N.IO_FORMAT, N.IO_VERSION
    b = bytearray(g); b[0] = ord("X"); _expect_io(N, b, FMT, 0)
    b = bytearray(g); b[4] = 2; _expect_io(N, b, VER, 4)
    b = bytearray(g); b[8] = 9; _expect_io(N, b, FMT, 8)
    b = bytearray(g); b[8] = 1; _expect_io(N, b, FMT, 8)
    for cut in (0, 3, 7, 15, 40, 47, 50, 60, 70, 88):
        _expect_io(N, g[:cut], FMT, None, "truncated")
    b = bytearray(g); b[48:52] = np.float32(-1.0).tobytes(); _expect_io(N, b, FMT, 48)
    b = bytearray(g); b[52:56] = np.float32(0.0).tobytes(); _expect_io(N, b, FMT, 52)
    b = bytearray(g); b[76:88] = b[64:76]; _expect_io(N, b, FMT, 76)      # duplicate coordinate
    b = bytearray(g); b[80] = 7; _expect_io(N, b, FMT, 76)                # column out of range
    b = bytearray(g); b[56] = 5; _expect_io(N, b, FMT, 56)                # count > rows*cols
    _expect_io(N, g + b"\x00", FMT, 89, "trailing")
    b = bytearray(g); b[32:40] = bytes(8); _expect_io(N, b, FMT, 32)      # zero rows
    with pytest.raises(N.IoError):
        N.decode_quantized(b"")


def test_encoder_validates_its_input(N, O):
    """test_io.cpp:251-270"""
    q = _artifact(N, O, 17, 9, 4, 9)
    assert len(q.outliers) >= 2
    import dataclasses
    bad = dataclasses.replace(q, scales=q.scales[:-1].copy())
    with pytest.raises(N.InvalidArgument):
        N.encode_quantized(bad)
    bad = dataclasses.replace(q, packed=q.packed[:-1].copy())
    with pytest.raises(N.InvalidArgument):
        N.encode_quantized(bad)
    s = q.scales.copy(); s[0] = -1.0
    with pytest.raises(N.InvalidArgument):
        N.encode_quantized(dataclasses.replace(q, scales=s))
    o = q.outliers.copy(); o[[0, -1]] = o[[-1, 0]]
    with pytest.raises(N.InvalidArgument):
        N.encode_quantized(dataclasses.replace(q, outliers=o))
    o = np.concatenate([q.outliers, np.array([(q.rows, 0, 1.0)], dtype=q.outliers.dtype)])
    with pytest.raises(N.InvalidArgument):
        N.encode_quantized(dataclasses.replace(q, outliers=o))


def test_wide_code_out_of_span_is_invalid_argument(N, O):
    q = _artifact(N, O, 5, 4, 3, 3)
    b = bytearray(N.encode_quantized(q))
    b[-1] = 200  # k=3 level byte beyond the span (unpack_levels)
    with pytest.raises(N.InvalidArgument):
        N.decode_quantized(bytes(b))


@pytest.mark.parametrize("rows,cols,bits,seed", [(17, 9, 4, 1), (64, 33, 3, 2), (7, 128, 8, 3),
                                                 (1, 1, 4, 4), (3, 5, 2, 5)])
def test_encode_matches_compiled_reference(N, O, R, rows, cols, bits, seed):
    q = _artifact(N, O, rows, cols, bits, seed, n_out=min(3, rows * cols))
    ours = N.encode_quantized(q)
    ref = R.make_quantized(rows, cols, bits, q.packed, q.scales, q.outliers, q.mean, q.stddev,
                           q.sigma_n).encode()
    assert ours == ref


def test_decode_errors_match_compiled_reference(N, O, R):
    """Random single-byte corruptions and truncations: same accept/reject
    decision, category and byte offset as the reference decoder."""
    q = _artifact(N, O, 6, 5, 4, 11, n_out=4)
    good = N.encode_quantized(q)
    rng = np.random.default_rng(0)
    cases = [good[:k] for k in range(0, len(good), 3)]
    for _ in range(300):
        b = bytearray(good)
        i = int(rng.integers(0, len(b)))
        b[i] = int(rng.integers(0, 256))
        cases.append(bytes(b))
    for b in cases:
        try:
            rq = R.decode(b)
            ref = ("ok", rq.packed.tobytes(), rq.outliers.tobytes())
        except R.RefError as e:
            ref = ("err", e.code, getattr(e, "offset", None))
        try:
            oq = N.decode_quantized(b)
            ours = ("ok", oq.packed.tobytes(), oq.outliers.tobytes())
        except N.IoError as e:
            ours = ("err", e.code, e.index)
        except N.InvalidArgument as e:
            ours = ("err", 9, None)
        if ref[0] == "err" and ref[1] == 9:
            ref = ("err", 9, None)  # std::exception (not io_error): offset not reported
        assert ours == ref, (b.hex(), ours, ref)


def test_zero_copy_views_keep_their_owner_alive(N, O):
    """decode_quantized returns zero-copy views of library memory: a kept
    array must stay valid after its QuantizedWeight is dropped, even when the
    next decode of the same size reuses the allocator's free block."""
    import gc
    import pickle
    a = _artifact(N, O, 64, 32, 4, 11, n_out=5)
    b = _artifact(N, O, 64, 32, 4, 12, n_out=5)
    q = N.decode_quantized(N.encode_quantized(a))
    kept_packed, kept_scales, kept_out = q.packed, q.scales, q.outliers
    ref = (kept_packed.copy(), kept_scales.copy(), kept_out.copy())
    del q
    gc.collect()
    others = [N.decode_quantized(N.encode_quantized(b)) for _ in range(4)]
    assert np.array_equal(kept_packed, ref[0])
    assert np.array_equal(kept_scales, ref[1])
    assert np.array_equal(kept_out, ref[2])
    # artifacts pickle as plain arrays (the multi-process driver ships them)
    back = pickle.loads(pickle.dumps(others[0]))
    assert np.array_equal(back.packed, others[0].packed) and back._owner is None

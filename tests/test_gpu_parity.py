"""GPU parity: the sm_100a product path (through the C ABI) against the CPU oracle.

Bit-exact for every byte of the archive and every bit of the decoded values.
Test cases follow the reference's own suites (proj/tests/test_chunk_codec.cpp,
test_container.cpp, test_pipeline.cpp, acceptance.cpp).
"""
import numpy as np
import pytest
import torch

from paper_2511_04140_b200 import F32, F64, CorruptError, FalconError, synth

pytestmark = pytest.mark.gpu

KINDS = ["walk", "decimal", "signflip", "outlier", "bits", "mixed"]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8).tobytes()


def gpu_archive(codec, vals, n, bv):
    arc, nb = codec.compress_device(dev(vals), chunk_n=n, batch_values=bv)
    return arc, nb, arc[:nb].cpu().numpy().tobytes()


# ---- golden vectors (test_chunk_codec.cpp:32-70, 216-227; FORMAT.md:106-123) ----
def test_golden_zero_chunk(codec):
    assert codec.compress_chunk(np.zeros(1025)) == bytes(11)
    assert codec.compress_chunk(np.zeros(1025, np.float32)) == bytes(7)


def test_golden_constant_chunk(codec):
    assert codec.compress_chunk(np.full(1025, 2.5)) == bytes([1, 2, 25] + [0] * 8)
    assert codec.compress_chunk(np.full(1025, 2.5, np.float32)) == bytes([1, 2, 25, 0, 0, 0, 0])


def test_golden_spike_chunk(codec):
    v = np.zeros(65)
    v[0] = 2.5
    golden = bytes.fromhex("010219000000000000000600808080800000008080")
    enc = codec.compress_chunk(v)
    assert enc == golden
    assert bits(codec.decompress_chunk(enc, 65, 65)) == bits(v)


def test_specials_take_raw_path(codec, oracle):
    vals = np.array([1.0, -0.0, np.nan, np.inf, -np.inf, 5e-324, 9.110900773177071, 1.25, 0.0,
                     np.frombuffer(np.uint64(0x7ff4000000000001).tobytes(), np.float64)[0],
                     np.frombuffer(np.uint64(0xfff8000000000123).tobytes(), np.float64)[0], -2.5, 1e300])
    padded = np.zeros(65)
    padded[: len(vals)] = vals
    enc = codec.compress_chunk(padded)
    assert enc[:2] == bytes([23, 16])
    assert enc == oracle.compress_chunk(padded)
    assert bits(codec.decompress_chunk(enc, 65, len(vals))) == bits(vals)


# ---- archives across kinds, precisions and geometries ----
@pytest.mark.parametrize("prec", [F64, F32])
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("n,bv,count", [(65, 1000, 5000), (257, 257 * 3, 4000), (1025, 1025 * 4, 30000),
                                         (1025, 1025 * 4096, 9000), (2049, 5000, 12000), (4097, 9000, 20000)])
def test_archive_parity_and_round_trip(codec, oracle, prec, kind, n, bv, count):
    vals = synth(kind, count, prec, dp=2 if prec == F64 else 1, seed=7 + count, period=100, block=n)
    want = oracle.compress_archive(vals, n, bv)
    arc, nb, got = gpu_archive(codec, vals, n, bv)
    assert got == want
    back = codec.decompress_device(arc, nb).cpu().numpy()
    assert bits(back) == bits(vals)


@pytest.mark.parametrize("prec", [F64, F32])
def test_gpu_decodes_cpu_archives(codec, oracle, prec):
    vals = synth("walk", 50000, prec, seed=3)
    arc = oracle.compress_archive(vals, 1025, 1025 * 8)
    t = torch.frombuffer(bytearray(arc), dtype=torch.uint8).cuda()
    back = codec.decompress_device(t, len(arc)).cpu().numpy()
    assert bits(back) == bits(vals)


def test_empty_input(codec):
    arc, nb = codec.compress_device(torch.empty(0, dtype=torch.float64, device="cuda"))
    assert nb == 47
    hdr = arc[:47].cpu().numpy().tobytes()
    assert hdr[:8] == b"FALCONA\0"
    assert codec.decompress_device(arc, nb).numel() == 0


def test_per_chunk_random_vs_oracle(codec, oracle):
    rng = np.random.default_rng(5)
    for n in (65, 257, 1025):
        for kind in KINDS:
            v = synth(kind, n, F64, seed=int(rng.integers(1 << 30)), block=n)
            enc = codec.compress_chunk(v)
            assert enc == oracle.compress_chunk(v)
            assert bits(codec.decompress_chunk(enc, n, n)) == bits(v)


# ---- corruption: same exception class and message as the reference ----
def _oracle_err(oracle, fn):
    try:
        fn()
    except Exception as e:  # noqa: BLE001
        return e
    return None


def test_chunk_corruption_matches_oracle(codec, oracle):
    rng = np.random.default_rng(33)
    vals = (rng.integers(0, 200001, 65) - 100000) / 1000.0
    enc = codec.compress_chunk(vals)
    cases = [enc[:k] for k in range(len(enc))] + [enc + b"\0"]
    bad_w = bytearray(enc); bad_w[10] = 65
    bad_meta = bytearray(enc); bad_meta[0] = 23
    bad_meta2 = bytearray(enc); bad_meta2[0] = 24; bad_meta2[1] = 16
    cases += [bytes(bad_w), bytes(bad_meta), bytes(bad_meta2)]
    for c in cases:
        e_cpu = _oracle_err(oracle, lambda: oracle.decompress_chunk(c, 65, 65))
        assert e_cpu is not None
        with pytest.raises(CorruptError) as ei:
            codec.decompress_chunk(c, 65, 65)
        assert str(ei.value) == e_cpu.message
    with pytest.raises(FalconError):
        codec.decompress_chunk(enc, 65, 66)


def test_flag_padding_rejected(codec):
    v = np.zeros(65)
    v[0] = 2.5
    enc = bytearray(codec.compress_chunk(v))
    enc[11] |= 0x40
    with pytest.raises(CorruptError, match="nonzero flag padding bits"):
        codec.decompress_chunk(bytes(enc), 65, 65)


def test_archive_corruption_messages(codec, oracle):
    vals = synth("walk", 3 * 1025 * 2 + 100, F64, seed=9)
    arc = oracle.compress_archive(vals, 1025, 1025 * 2)
    variants = {
        "trailing": arc + b"\x00",
        "truncated": arc[:-5],
        "bad_count": arc[:47] + (3).to_bytes(4, "little") + arc[51:],
    }
    # a corrupt chunk in batch 1
    first = 47 + 4 + 4 * 2 + int.from_bytes(arc[51:55], "little") + int.from_bytes(arc[55:59], "little")
    off1 = first + 4 + 4 * 2
    mod = bytearray(arc)
    mod[off1 + 10] = 70  # w > 64
    variants["bad_chunk"] = bytes(mod)
    for name, a in variants.items():
        e_cpu = _oracle_err(oracle, lambda: oracle.decompress_archive(a, F64))
        assert e_cpu is not None, name
        t = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
        with pytest.raises(CorruptError) as ei:
            codec.decompress_device(t, len(a))
        assert str(ei.value) == e_cpu.message, name


def test_precision_mismatch(codec):
    vals = synth("walk", 2000, F64)
    arc, nb = codec.compress_device(dev(vals))
    with pytest.raises(FalconError, match="archive precision does not match the requested value type"):
        codec.decompress_device(arc, nb, dtype=torch.float32)


# ---- host-resident pipeline (test_pipeline.cpp:124-216) ----
@pytest.mark.parametrize("streams,workers", [(1, 1), (2, 3), (16, 0)])
def test_pipeline_bytes_independent_of_streams(codec, oracle, streams, workers):
    from paper_2511_04140_b200 import options
    vals = synth("walk", 5 * 1025 + 400, F64, seed=17)
    want = oracle.compress_archive(vals, 1025, 2 * 1025)
    opt = options(1025, 2 * 1025, streams, workers)
    got = codec.compress_host(vals, opt).tobytes()
    assert got == want
    back = codec.decompress_host(got, F64, opt)
    assert bits(back) == bits(vals)


def test_pipeline_stream_callbacks(codec, oracle):
    from paper_2511_04140_b200 import PipelineStats, options
    vals = synth("outlier", 40000, F64, seed=2, period=100)
    pos = [0]

    def read(maxv):
        k = min(maxv, 777, len(vals) - pos[0])
        out = vals[pos[0]: pos[0] + k]
        pos[0] += k
        return out

    archive = bytearray()

    def store(off, b):
        if len(archive) < off + len(b):
            archive.extend(b"\0" * (off + len(b) - len(archive)))
        archive[off: off + len(b)] = b

    st = PipelineStats()
    codec.compress_stream(read, store, F64, options(1025, 1025 * 3, 4, 2), st)
    assert bytes(archive) == oracle.compress_archive(vals, 1025, 1025 * 3)
    assert st.values == len(vals) and st.batches == (len(vals) + 3074) // 3075
    got = np.zeros_like(vals)

    def put(first, v):
        got[first: first + len(v)] = v

    codec.decompress_stream(bytes(archive), put, F64, options(1025, 1025 * 3, 3, 2))
    assert bits(got) == bits(vals)


# ---- full-size properties (BASELINE configs at reduced count where the oracle is slow) ----
def test_large_outlier_round_trip_and_ratio(codec, oracle):
    n = 16 * 4198400  # 16 full batches of cfg2's kind
    vals = synth("outlier", n, F64, dp=2, seed=1, period=100)
    arc, nb = codec.compress_device(dev(vals))
    back = codec.decompress_device(arc, nb)
    assert torch.equal(back.view(torch.int64), dev(vals).view(torch.int64))
    ratio = nb / vals.nbytes
    assert 0.13 < ratio < 0.16
    # spot-check one batch against the oracle byte for byte
    sub = vals[: 4198400]
    want = oracle.compress_archive(sub, 1025, 4198400)
    a2, n2 = codec.compress_device(dev(sub))
    assert a2[:n2].cpu().numpy().tobytes() == want


def test_unsupported_chunk_n_fails_loudly(codec):
    with pytest.raises(FalconError, match="not supported"):
        codec.compress_device(dev(np.zeros(9000)), chunk_n=8193, batch_values=9000)


def test_chained_device_round_trip_without_host_sync(codec, oracle):
    # compress_device_async leaves the archive length on the device; the chained decoder
    # reads it there, so the pair runs back to back on one stream
    from paper_2511_04140_b200 import compress_bound, read_header
    vals = synth("outlier", 200_000, F64, dp=2, seed=41, period=100)
    want = oracle.compress_archive(vals, 1025, 1025 * 16)
    d = dev(vals)
    arc = torch.empty(compress_bound(F64, len(vals), 1025, 1025 * 16), dtype=torch.uint8, device="cuda")
    d_nb = torch.zeros(1, dtype=torch.int64, device="cuda")
    back = torch.empty_like(d)
    info = read_header(want[:47])
    for _ in range(3):
        back.zero_()
        codec.compress_device_async(d, arc, d_nb, 1025, 1025 * 16)
        codec.decompress_device_chained(arc, d_nb, info, back)
    codec.sync()
    assert int(d_nb.item()) == len(want)
    assert arc[: len(want)].cpu().numpy().tobytes() == want
    assert bits(back.cpu().numpy()) == bits(vals)


@pytest.mark.parametrize("shift", [1, 3, 8, 13])
def test_decode_from_unaligned_archive(codec, oracle, shift):
    # the archive need not start on a 16-B boundary: staging, the frame walker and the
    # vector loads all fall back to byte-exact paths
    vals = synth("outlier", 3 * 1025 * 8 + 77, F64, dp=2, seed=9, period=100)
    arc = oracle.compress_archive(vals, 1025, 1025 * 8)
    buf = torch.zeros(len(arc) + 16, dtype=torch.uint8, device="cuda")
    buf[shift:shift + len(arc)] = torch.frombuffer(bytearray(arc), dtype=torch.uint8).cuda()
    back = codec.decompress_device(buf[shift:shift + len(arc)], len(arc)).cpu().numpy()
    assert bits(back) == bits(vals)

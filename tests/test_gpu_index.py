"""Batch-offset index and random-access decode.  The format has no
batch index (FORMAT.md:10-14); falcon_archive_index walks the frames once on the device
(read_batch, container.cpp:113-132) and falcon_decompress_device_range decodes any batch
range from it, bit-exactly, with the decoder's validation and absolute batch numbers."""
import numpy as np
import pytest
import torch

from paper_2511_04140_b200 import F32, F64, CorruptError, synth

pytestmark = pytest.mark.gpu


def frame_starts(archive: bytes):
    """Reference frame walk on the host (container.cpp:113-132)."""
    n_batches = int.from_bytes(archive[31:39], "little")
    cur, out = 47, []
    for _ in range(n_batches):
        out.append(cur)
        cnt = int.from_bytes(archive[cur:cur + 4], "little")
        sizes = np.frombuffer(archive[cur + 4:cur + 4 + 4 * cnt], dtype="<u4")
        cur += 4 + 4 * cnt + int(sizes.sum())
    return out + [cur]


@pytest.mark.parametrize("prec", [F64, F32])
def test_index_and_random_batch_ranges(codec, oracle, prec):
    bv = 1025 * 3 + 17
    vals = synth("outlier", 40 * bv + 1234, prec, dp=2 if prec == F64 else 1, seed=5, period=100)
    arc_bytes = oracle.compress_archive(vals, 1025, bv)
    arc = torch.frombuffer(bytearray(arc_bytes), dtype=torch.uint8).cuda()
    idx = codec.archive_index(arc, len(arc_bytes))
    assert list(idx) == frame_starts(arc_bytes)
    rng = np.random.default_rng(1)
    nb = len(idx) - 1
    for first, count in [(0, nb), (nb - 1, 1), (0, 1), (7, 5)] + [tuple(sorted(rng.integers(0, nb, 2))) for _ in range(6)]:
        count = max(count - first, 1) if count > first else 1
        count = min(count, nb - first)
        got = codec.decompress_range(arc, idx, first, count).cpu().numpy()
        want = vals[first * bv:min((first + count) * bv, len(vals))]
        assert got.tobytes() == want.tobytes(), (first, count)


def test_range_decode_reports_absolute_batch_numbers(codec, oracle):
    bv = 2050
    vals = synth("walk", 20 * bv, F64, seed=3)
    arc_bytes = bytearray(oracle.compress_archive(vals, 1025, bv))
    idx = frame_starts(bytes(arc_bytes))
    # corrupt the first chunk header of batch 12: alpha/beta bytes become an invalid pair
    chunk0 = idx[12] + 4 + 4 * 2
    arc_bytes[chunk0] = 30
    arc_bytes[chunk0 + 1] = 0
    arc = torch.frombuffer(arc_bytes, dtype=torch.uint8).cuda()
    with pytest.raises(CorruptError, match=r"\(batch 12\)"):
        codec.decompress_range(arc, np.array(idx, np.uint64), 10, 5)
    # batches before the damage still decode
    got = codec.decompress_range(arc, np.array(idx, np.uint64), 3, 9).cpu().numpy()
    assert got.tobytes() == vals[3 * bv:12 * bv].tobytes()


def test_index_rejects_truncated_archive(codec, oracle):
    vals = synth("walk", 30000, F64, seed=4)
    arc_bytes = oracle.compress_archive(vals, 1025, 4100)
    cut = torch.frombuffer(bytearray(arc_bytes[:-100]), dtype=torch.uint8).cuda()
    with pytest.raises(CorruptError):
        codec.archive_index(cut, len(arc_bytes) - 100)

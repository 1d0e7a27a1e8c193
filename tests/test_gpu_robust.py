"""Robustness of the device path against crafted archives and misuse, each compared with
the CPU oracle's error class and message where the reference defines one:

* size tables whose u32 entries sum past 2^32 (read_batch sums in u64,
  container.cpp:124-128) and entries larger than any valid chunk;
* the " (batch N)" suffix on errors surfaced by falcon_ctx_sync after async decodes
  (pipeline.hpp:404-405, 415-416);
* an output buffer too small for the archive on the async compress -> chained decode
  path: a clean capacity error, no out-of-bounds reads, the context stays usable.
"""
import numpy as np
import pytest
import torch

from paper_2511_04140_b200 import F64, CorruptError, FalconError, compress_bound, read_header, synth

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8).tobytes()


def oracle_message(oracle, arc, prec=F64):
    try:
        oracle.decompress_archive(arc, prec)
    except Exception as e:  # noqa: BLE001
        return e.message
    return None


def gpu_message(codec, arc):
    t = torch.frombuffer(bytearray(arc), dtype=torch.uint8).cuda()
    with pytest.raises(CorruptError) as ei:
        codec.decompress_device(t, len(arc))
    return str(ei.value)


def frame_tables(arc, n_chunks):
    """(count offset, [entry offsets]) of batch 0."""
    return 47, [51 + 4 * i for i in range(n_chunks)]


def test_size_table_wrapping_past_2_32(codec, oracle):
    vals = synth("walk", 1025 * 4, F64, seed=3)
    arc = bytearray(oracle.compress_archive(vals, 1025, 1025 * 4))
    _, ent = frame_tables(arc, 4)
    s = [int.from_bytes(arc[o:o + 4], "little") for o in ent]
    # entries summing to 2^32 + sum(s): a u32 sum would wrap to exactly the true payload
    arc[ent[0]:ent[0] + 4] = (0xFFFFFFFF).to_bytes(4, "little")
    arc[ent[1]:ent[1] + 4] = ((s[0] + s[1] + 1) & 0xFFFFFFFF).to_bytes(4, "little")
    want = oracle_message(oracle, bytes(arc))
    assert want is not None and "batch payload truncated" in want
    assert gpu_message(codec, bytes(arc)) == want


def test_oversize_entry_inside_the_archive(codec, oracle):
    # incompressible chunks (~8.2 KB each); entry 0 takes chunk 1's bytes too, entry 1 = 0:
    # the payload total is unchanged, chunk 0 is longer than any valid chunk
    vals = synth("bits", 1025 * 8, F64, seed=5)
    arc = bytearray(oracle.compress_archive(vals, 1025, 1025 * 8))
    _, ent = frame_tables(arc, 8)
    s = [int.from_bytes(arc[o:o + 4], "little") for o in ent]
    arc[ent[0]:ent[0] + 4] = (s[0] + s[1]).to_bytes(4, "little")
    arc[ent[1]:ent[1] + 4] = (0).to_bytes(4, "little")
    want = oracle_message(oracle, bytes(arc))
    assert want is not None
    assert gpu_message(codec, bytes(arc)) == want
    # and with the entries moved within the payload (chunk 3 takes 4's bytes)
    arc2 = bytearray(oracle.compress_archive(vals, 1025, 1025 * 8))
    arc2[ent[3]:ent[3] + 4] = (s[3] + s[4]).to_bytes(4, "little")
    arc2[ent[4]:ent[4] + 4] = (0).to_bytes(4, "little")
    want2 = oracle_message(oracle, bytes(arc2))
    assert want2 is not None
    assert gpu_message(codec, bytes(arc2)) == want2


def test_async_decode_error_has_batch_suffix(codec, oracle):
    vals = synth("walk", 3 * 1025 * 2 + 100, F64, seed=9)
    arc = bytearray(oracle.compress_archive(vals, 1025, 1025 * 2))
    first = 47 + 4 + 4 * 2 + int.from_bytes(arc[51:55], "little") + int.from_bytes(arc[55:59], "little")
    arc[first + 4 + 4 * 2 + 10] = 70     # batch 1, chunk 0: w > 64
    want = oracle_message(oracle, bytes(arc))
    assert want.endswith("(batch 1)")
    info = read_header(bytes(arc[:47]))
    t = torch.frombuffer(bytearray(arc), dtype=torch.uint8).cuda()
    out = torch.empty(len(vals), dtype=torch.float64, device="cuda")
    codec.decompress_device_async(t, len(arc), info, out)
    with pytest.raises(CorruptError) as ei:
        codec.sync()
    assert str(ei.value) == want
    codec.sync()    # the error words were reset


def test_capacity_overflow_on_the_chained_path(codec, oracle):
    vals = synth("bits", 1025 * 64, F64, seed=6)        # incompressible: archive ~ input size
    d = torch.from_numpy(vals).cuda()
    need = compress_bound(F64, len(vals), 1025, 1025 * 16)
    small = torch.zeros(need // 3, dtype=torch.uint8, device="cuda")
    d_nb = torch.zeros(1, dtype=torch.int64, device="cuda")
    want = oracle.compress_archive(vals, 1025, 1025 * 16)
    info = read_header(want[:47])
    back = torch.empty_like(d)
    codec.compress_device_async(d, small, d_nb, 1025, 1025 * 16)
    codec.decompress_device_chained(small, d_nb, info, back)
    with pytest.raises(FalconError, match="output capacity too small"):
        codec.sync()
    assert int(d_nb.item()) == 0          # no length past the buffer is published
    # the context is still healthy
    arc, nb = codec.compress_device(d, 1025, 1025 * 16)
    assert arc[:nb].cpu().numpy().tobytes() == want
    assert bits(codec.decompress_device(arc, nb).cpu().numpy()) == bits(vals)


@pytest.mark.parametrize("kind,prec", [("walk", F64), ("outlier", F64), ("mixed", 1)])
def test_random_corruption_fuzz_matches_oracle(codec, oracle, kind, prec):
    # mutations of a multi-batch archive (byte flips anywhere after the header, truncations,
    # inserted bytes): the device decoder either fails with the oracle's exact error text
    # or returns the oracle's exact values (test_oracle_vs_ref.py:36 does this CPU-side)
    vals = synth(kind, 5 * 1025 * 3 + 211, prec, seed=21, period=100)
    arc = oracle.compress_archive(vals, 1025, 1025 * 3)
    rng = np.random.default_rng(77 + prec)
    for trial in range(150):
        a = bytearray(arc)
        r = trial % 5
        if r == 0:
            a = a[: int(rng.integers(47, len(a)))]
        elif r == 1:
            pos = int(rng.integers(47, len(a)))
            a[pos:pos] = bytes([int(rng.integers(0, 256))])
        else:
            for _ in range(1 + r // 3):
                pos = int(rng.integers(47, len(a)))
                a[pos] ^= int(rng.integers(1, 256))
        a = bytes(a)
        try:
            want_vals = oracle.decompress_archive(a, prec)
            want_msg = None
        except Exception as e:  # noqa: BLE001
            want_vals, want_msg = None, e.message
        t = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
        if want_msg is None:
            got = codec.decompress_device(t, len(a)).cpu().numpy()
            assert bits(got) == bits(want_vals), f"trial {trial}: values differ"
        else:
            with pytest.raises(FalconError) as ei:
                codec.decompress_device(t, len(a))
            assert str(ei.value) == want_msg, f"trial {trial}"


def test_sync_error_does_not_leak_into_the_next_call(codec, oracle):
    # a synchronous call that fails leaves its device error word cleared: the next call on
    # the same context (and falcon_ctx_sync) reports only its own outcome
    vals = synth("outlier", 1025 * 8 + 7, F64, seed=21, period=100)
    arc = oracle.compress_archive(vals, 1025, 1025 * 4)
    bad = torch.frombuffer(bytearray(arc[:-9]), dtype=torch.uint8).cuda()
    with pytest.raises(CorruptError):
        codec.decompress_device(bad, len(arc) - 9)
    d = torch.from_numpy(vals).cuda()
    got, nb = codec.compress_device(d, chunk_n=1025, batch_values=1025 * 4)
    assert got[:nb].cpu().numpy().tobytes() == arc
    codec.sync()
    back = codec.decompress_device(got, nb).cpu().numpy()
    assert bits(back) == bits(vals)

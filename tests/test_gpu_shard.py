"""Multi-GPU data path on one GPU: every batch-range shard is compressed
on the device independently, the shards are assembled after the single offset exchange
(here: the list of shard byte totals), and the result is byte-identical to the archive of
the whole stream -- the CPU oracle's (container.cpp:88-111: frames are context-free).
Each shard's frames then decode on the device into its own value range."""
import numpy as np
import pytest
import torch

from paper_2511_04140_b200 import F32, F64, shard, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec,world", [(F64, 2), (F64, 3), (F32, 4)])
def test_sharded_archive_matches_whole_stream(codec, oracle, prec, world):
    n, bv = 61 * 1025 * 4 + 999, 1025 * 4
    vals = synth("outlier", n, prec, dp=2 if prec == F64 else 1, seed=17, period=100)
    want = oracle.compress_archive(vals, 1025, bv)
    plans = shard.plan_shards(n, bv, world)
    d = torch.from_numpy(vals).cuda()
    parts, totals = [], []
    for s in plans:
        arc, nb = codec.compress_device(d[s.first_value:s.first_value + s.n_values], 1025, bv)
        parts.append(arc[:nb].cpu().numpy().tobytes())
        totals.append(nb - shard.HEADER_BYTES)
    offsets = shard.shard_offsets(totals)                      # the one exchange step
    whole = shard.assemble(prec, 1025, bv, n, parts)
    assert whole == want
    assert offsets[-1] + totals[-1] == len(want)
    back = torch.empty_like(d)
    for s, p, off in zip(plans, parts, offsets):
        # each rank decodes its frames (global archive bytes [off, off + total)) by itself
        frames = shard.global_header(prec, 1025, bv, s.n_values) + whole[off:off + len(p) - shard.HEADER_BYTES]
        assert frames == p
        dev_arc = torch.frombuffer(bytearray(frames), dtype=torch.uint8).cuda()
        codec.decompress_device(dev_arc, len(frames), out=back[s.first_value:s.first_value + s.n_values])
    assert back.cpu().numpy().tobytes() == vals.tobytes()

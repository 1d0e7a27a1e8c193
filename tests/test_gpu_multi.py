"""Multi-GPU paths of the product (SURVEY.md 8b "device list", 8e batch-range shards):

* falcon_compress_host_multi / falcon_decompress_host_multi with 1-3 contexts (on the one
  GPU of the test box each context is its own stream set and scratch; on a multi-GPU box
  one per device): bytes equal the single-GPU archive and the oracle's, round trips are
  bit-exact, corrupt archives fail with the reference's message;
* two processes, each with its own CUDA context, run the sharded data path: compress its
  batch range on the GPU, all-gather the frame byte totals over gloo (the one exchange),
  rank 0 assembles the global archive (47-byte header + frames in rank order), then every
  rank decodes its own batch range straight out of the global archive through the device
  batch index (falcon_archive_index + falcon_decompress_device_range).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_04140_b200 import (F32, F64, Codec, CorruptError, compress_host_multi, decompress_host_multi,
                                   options, shard, synth)

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8).tobytes()


@pytest.mark.parametrize("n_ctx", [1, 2, 3])
@pytest.mark.parametrize("prec", [F64, F32])
def test_host_multi_equals_single_gpu_archive(codec, oracle, n_ctx, prec):
    vals = synth("outlier" if prec == F64 else "mixed", 9 * 3 * 1025 + 500, prec, seed=5, period=100)
    opt = options(1025, 3 * 1025, 4, 2)
    want = oracle.compress_archive(vals, 1025, 3 * 1025)
    codecs = [codec] + [Codec(0) for _ in range(n_ctx - 1)]
    got = compress_host_multi(codecs, vals, opt).tobytes()
    assert got == want
    assert got == codec.compress_host(vals, opt).tobytes()
    back = decompress_host_multi(codecs, got, prec, opt)
    assert bits(back) == bits(vals)


def test_host_multi_corrupt_archive_message(codec, oracle):
    vals = synth("walk", 6 * 1025 * 2 + 7, F64, seed=8)
    arc = bytearray(oracle.compress_archive(vals, 1025, 2 * 1025))
    variants = {"trailing": bytes(arc) + b"\0", "truncated": bytes(arc[:-3])}
    codecs = [codec, Codec(0)]
    for name, a in variants.items():
        try:
            oracle.decompress_archive(a, F64)
            want = None
        except Exception as e:  # noqa: BLE001
            want = e.message
        with pytest.raises(CorruptError) as ei:
            decompress_host_multi(codecs, a, F64, options(1025, 2 * 1025, 2, 1))
        assert str(ei.value) == want, name


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


N_VALUES = 11 * 4 * 1025 + 321
BV = 4 * 1025


def _rank_main(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    codec = Codec(0)                              # this rank's own CUDA context
    vals = synth("field", N_VALUES, F64, dp=2, seed=3)
    sh = shard.plan_shards(N_VALUES, BV, world)[rank]
    # this rank's batch range, generated on its device (counter-based field)
    d = torch.empty(sh.n_values, dtype=torch.float64, device="cuda")
    codec.synth_device(d, "field", first=sh.first_value, dp=2, seed=3)
    assert bits(d.cpu().numpy()) == bits(vals[sh.first_value:sh.first_value + sh.n_values])
    arc, nb = codec.compress_device(d, 1025, BV)
    local = arc[:nb].cpu().numpy().tobytes()
    totals = shard.exchange_frame_bytes(nb - shard.HEADER_BYTES)      # the one exchange
    offs = shard.shard_offsets(totals)
    parts = [None] * world
    dist.all_gather_object(parts, local[shard.HEADER_BYTES:])
    whole = shard.global_header(F64, 1025, BV, N_VALUES) + b"".join(parts)
    assert len(whole) == offs[-1] + totals[-1]
    if rank == 0:
        with open(os.path.join(out_dir, "global.fln"), "wb") as f:
            f.write(whole)
    # decode this rank's batch range out of the GLOBAL archive via the device index
    g = torch.frombuffer(bytearray(whole), dtype=torch.uint8).cuda()
    idx = codec.archive_index(g, len(whole))
    back = codec.decompress_range(g, idx, sh.first_batch, sh.n_batches).cpu().numpy()
    ok = bits(back) == bits(vals[sh.first_value:sh.first_value + sh.n_values])
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    if rank == 0:
        with open(os.path.join(out_dir, "ok.txt"), "w") as f:
            f.write(" ".join(str(x) for x in flags))
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_run_the_sharded_product(tmp_path, oracle):
    mp.spawn(_rank_main, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    assert open(tmp_path / "ok.txt").read() == "True True"
    vals = synth("field", N_VALUES, F64, dp=2, seed=3)
    assert open(tmp_path / "global.fln", "rb").read() == oracle.compress_archive(vals, 1025, BV)


# ---- files through GPU-direct storage (falcon_compress_file / falcon_decompress_file) ----
@pytest.mark.parametrize("prec,kind", [(F64, "outlier"), (F32, "mixed")])
def test_file_round_trip_through_gds(codec, oracle, tmp_path, prec, kind):
    from paper_2511_04140_b200 import options as opts
    vals = synth(kind, 33 * 1025 * 4 + 91, prec, seed=12, period=100)
    raw, fln, back = tmp_path / "v.raw", tmp_path / "v.fln", tmp_path / "back.raw"
    vals.tofile(raw)
    nb, io = codec.compress_file(str(raw), str(fln), prec, opts(1025, 4 * 1025, 4, 0))
    want = oracle.compress_archive(vals, 1025, 4 * 1025)
    assert open(fln, "rb").read() == want and nb == len(want)
    nv, io2 = codec.decompress_file(str(fln), str(back), prec)
    assert nv == len(vals) and open(back, "rb").read() == vals.tobytes()
    assert io in (0, 1) and io2 in (0, 1)
    # a truncated archive fails like the reference
    (tmp_path / "t.fln").write_bytes(want[:-9])
    with pytest.raises(CorruptError):
        codec.decompress_file(str(tmp_path / "t.fln"), str(tmp_path / "t.raw"), prec)

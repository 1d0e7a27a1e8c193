"""CPU, world_size 2 over gloo: batch-range sharding + the one offset exchange produce an
archive byte-identical to the single-process one (shard archives come from the oracle;
the GPU path produces the same bytes per shard, see test_gpu_parity)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_04140_b200 import shard


def test_plan_covers_all_batches():
    for n, bv, g in [(10, 3, 2), (4198400 * 7 + 5, 4198400, 8), (0, 10, 4), (1, 10, 3)]:
        s = shard.plan_shards(n, bv, g)
        assert sum(x.n_values for x in s) == n
        assert all(s[i].first_value + s[i].n_values == s[i + 1].first_value for i in range(g - 1))
        assert all(x.first_value % bv == 0 for x in s if x.n_values)


def test_split_and_assemble_round_trip(oracle):
    vals = oracle.synth("outlier", 23 * 1000 + 17, seed=2, period=100)
    whole = oracle.compress_archive(vals, 1025, 1000 * 3)
    shards = shard.plan_shards(len(vals), 3000, 3)
    parts = shard.split_frames(whole, shards, 0)
    for s, p in zip(shards, parts):
        assert p == oracle.compress_archive(vals[s.first_value:s.first_value + s.n_values], 1025, 3000)
    assert shard.assemble(0, 1025, 3000, len(vals), parts) == whole


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    orc = Oracle()
    vals = orc.synth("walk", 40 * 1025 + 333, seed=4)
    bv = 4 * 1025
    sh = shard.plan_shards(len(vals), bv, world)[rank]
    local = orc.compress_archive(vals[sh.first_value:sh.first_value + sh.n_values], 1025, bv)
    totals = shard.exchange_frame_bytes(len(local) - shard.HEADER_BYTES)
    offs = shard.shard_offsets(totals)
    # each rank writes its frames at its offset of a shared file; rank 0 writes the header
    path = os.path.join(result_dir, "sharded.fln")
    dist.barrier()
    if rank == 0:
        with open(path, "wb") as f:
            f.write(shard.global_header(0, 1025, bv, len(vals)))
            f.truncate(offs[-1] + totals[-1])
    dist.barrier()
    with open(path, "r+b") as f:
        f.seek(offs[rank])
        f.write(local[shard.HEADER_BYTES:])
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_exchange(tmp_path, oracle):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    vals = oracle.synth("walk", 40 * 1025 + 333, seed=4)
    got = open(tmp_path / "sharded.fln", "rb").read()
    assert got == oracle.compress_archive(vals, 1025, 4 * 1025)
    back = oracle.decompress_archive(got)
    assert back.view(np.uint64).tobytes() == vals.view(np.uint64).tobytes()

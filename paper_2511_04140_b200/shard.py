"""Multi-GPU sharding of one archive by contiguous batch ranges.

Batch frames are context-free (container.cpp:88-111): frame b depends only on the values
of batch b.  So rank g of G compresses batches [floor(g*B/G), floor((g+1)*B/G)) as an
independent archive, and the global archive is the 47-byte header (container.cpp:44-55)
followed by every shard's frames in rank order.  The only exchange is one all-gather of
the G shard byte totals (an exclusive scan gives each shard's archive offset); on
NVSwitch that is one 8-byte NCCL collective.  Decompression needs no exchange: rank g
decodes its own frames into its own value range.
"""
from __future__ import annotations

from dataclasses import dataclass

HEADER_BYTES = 47


@dataclass(frozen=True)
class Shard:
    rank: int
    first_batch: int
    n_batches: int
    first_value: int
    n_values: int


def plan_shards(n_values: int, batch_values: int, world: int) -> list[Shard]:
    """Contiguous batch ranges per rank; the short final batch lands on the last rank."""
    if batch_values <= 0 or world <= 0:
        raise ValueError("batch_values and world must be positive")
    n_batches = (n_values + batch_values - 1) // batch_values
    shards = []
    for g in range(world):
        b0 = g * n_batches // world
        b1 = (g + 1) * n_batches // world
        v0 = min(b0 * batch_values, n_values)
        v1 = min(b1 * batch_values, n_values)
        shards.append(Shard(g, b0, b1 - b0, v0, v1 - v0))
    return shards


def shard_offsets(frame_bytes: list[int]) -> list[int]:
    """Archive offset of each shard's frames: 47 + exclusive scan of the frame totals."""
    out, acc = [], HEADER_BYTES
    for nb in frame_bytes:
        out.append(acc)
        acc += nb
    return out


def exchange_frame_bytes(local_frame_bytes: int, group=None, device=None) -> list[int]:
    """All-gather the per-rank frame byte totals (the single collective of the path)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.tensor([local_frame_bytes], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [int(x.item()) for x in out]


def global_header(precision: int, chunk_n: int, batch_values: int, n_values: int) -> bytes:
    """write_header (container.cpp:44-55) for the whole sharded stream."""
    n_batches = (n_values + batch_values - 1) // batch_values if batch_values else 0
    h = bytearray(b"FALCONA\0")
    h += (1).to_bytes(2, "little")
    h += bytes([precision])
    h += chunk_n.to_bytes(4, "little")
    h += batch_values.to_bytes(8, "little")
    h += n_values.to_bytes(8, "little")
    h += n_batches.to_bytes(8, "little")
    h += bytes(8)
    return bytes(h)


def assemble(precision: int, chunk_n: int, batch_values: int, n_values: int,
             shard_archives: list[bytes]) -> bytes:
    """Concatenate per-shard archives (each with its own 47-byte header) into one."""
    parts = [global_header(precision, chunk_n, batch_values, n_values)]
    parts += [a[HEADER_BYTES:] for a in shard_archives]
    return b"".join(parts)


def split_frames(archive: bytes, shards: list[Shard], precision: int) -> list[bytes]:
    """Cut a whole archive into per-shard archives by walking the frames
    (read_batch, container.cpp:113-132); each gets a header with its own counts."""
    chunk_n = int.from_bytes(archive[11:15], "little")
    bv = int.from_bytes(archive[15:23], "little")
    cursor = HEADER_BYTES
    starts = []
    n_batches = int.from_bytes(archive[31:39], "little")
    for _ in range(n_batches):
        starts.append(cursor)
        cnt = int.from_bytes(archive[cursor:cursor + 4], "little")
        table = archive[cursor + 4:cursor + 4 + 4 * cnt]
        payload = sum(int.from_bytes(table[4 * i:4 * i + 4], "little") for i in range(cnt))
        cursor += 4 + 4 * cnt + payload
    starts.append(cursor)
    out = []
    for s in shards:
        body = archive[starts[s.first_batch]:starts[s.first_batch + s.n_batches]]
        out.append(global_header(precision, chunk_n, bv, s.n_values) + body)
    return out

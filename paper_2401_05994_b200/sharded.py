"""Multi-GPU chunked compress / decompress (one process per GPU).

Restates the CLI's multiblock driver (``tools/mgrc.cpp:363-542``) over
``torch.distributed``: the array is planned into slabs by ``plan_chunks``
(``chunking.cpp:38-110``, slowest axis first); slab ``b`` of ``B`` belongs to
rank ``floor(b * G / B)``, so every rank owns a contiguous range of the input
rows and of the output stream.  The blocks are independent containers
(SPEC.md:478), so the only collectives are tiny:

  1. REL mode: all-gather of the per-rank ``[min, max]`` (INF); for S norms
     the file-order serial sum of squares of the CLI (``mgrc.cpp:197-233``)
     is chained rank to rank (one double each, exact) and all-gathered, so
     the global absolute tolerance is bit-identical (``mgrc.cpp:405-418``);
  2. all-gather of the per-block compressed sizes, from which every rank
     computes the absolute offsets ``4 + 8 B + sum(sizes before)`` of the
     multiblock stream ``u32 count | u64 offsets[count] | containers``
     (``mgrc.cpp:258-275``).

The resulting stream is byte-identical for any number of ranks and identical
to the CLI's (for S-REL with plans that split inner axes the per-rank sums
are combined in rank order instead — an ulp-level difference in tau).

``block_compress`` / ``block_stats`` default to the sm_100a library; the CPU
tests inject the oracle to exercise the host logic under ``gloo``.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import Codec, DType, ErrorSpec, Mode, Norm, MgrcError


def owner_of(block: int, nblocks: int, world: int) -> int:
    """Rank owning block ``block``: floor(b * G / B) (contiguous ranges)."""
    return (block * world) // nblocks


def blocks_of(rank: int, nblocks: int, world: int) -> List[int]:
    return [b for b in range(nblocks) if owner_of(b, nblocks, world) == rank]


def block_coords(ranges, coords: Sequence[np.ndarray]):
    return [np.asarray(coords[a][int(r[0]):int(r[1])], dtype=np.float64) for a, r in enumerate(ranges)]


def frame_header(sizes: Sequence[int]) -> bytes:
    """u32 count | u64 absolute offsets (mgrc.cpp:258-275)."""
    n = len(sizes)
    out = [struct.pack("<I", n)]
    off = 4 + 8 * n
    for s in sizes:
        out.append(struct.pack("<Q", off))
        off += s
    return b"".join(out)


@dataclass
class ShardedStream:
    """This rank's share of one multiblock stream."""

    header: bytes            # count + offset table (identical on every rank)
    sizes: List[int]         # every block's container size, plan order
    my_blocks: List[int]
    my_offset: int           # absolute offset of this rank's first container
    my_bytes: bytes          # this rank's containers, concatenated

    @property
    def total_len(self) -> int:
        return len(self.header) + sum(self.sizes)

    def write_into(self, buf) -> None:
        """Place this rank's part (and, on every rank, the header) in a buffer of total_len bytes."""
        mv = memoryview(buf)
        mv[: len(self.header)] = self.header
        mv[self.my_offset: self.my_offset + len(self.my_bytes)] = self.my_bytes


def _default_compress(block, grid_shape, coords, spec, codec):
    from . import compress, make_grid

    return compress(block, make_grid(grid_shape, coords), spec, codec)


def _default_stats(block):
    from . import field_stats

    mn, mx, nonfinite = field_stats(block)
    return mn, mx, nonfinite


def _default_sumsq(block, s0: float) -> float:
    from . import serial_sumsq

    return serial_sumsq(block, s0)


def compress_sharded(read_block: Callable[[int, list], object], shape: Sequence[int], dtype: DType,
                     spec: ErrorSpec, codec: Codec = Codec.huffman, chunk_mem: int = 0,
                     coords: Optional[Sequence[Sequence[float]]] = None, group=None,
                     block_compress=None, block_stats=None, block_sumsq=None) -> ShardedStream:
    """Chunked compress across the ranks of ``group`` (mgrc.cpp:363-484).

    ``read_block(b, ranges)`` returns block ``b`` (numpy or torch, host or
    device) for this rank's blocks only.
    """
    import torch.distributed as dist

    from . import plan_chunks

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    block_compress = block_compress or _default_compress
    block_stats = block_stats or _default_stats
    block_sumsq = block_sumsq or _default_sumsq
    shape = tuple(int(s) for s in shape)
    plan = plan_chunks(shape, dtype, chunk_mem if chunk_mem > 0 else (1 << 64) - 1)
    nb = plan.shape[0]
    mine = blocks_of(rank, nb, world)
    data = {b: read_block(b, plan[b].tolist()) for b in mine}

    if nb == 1:  # single block: the user's spec and grid, still framed (mgrc.cpp:389-404, :476)
        ucoords = None if coords is None else [np.asarray(c, dtype=np.float64) for c in coords]
        blob = block_compress(data[0], shape, ucoords, spec, codec) if mine else b""
        sizes = _allgather_ints([len(blob)] if mine else [], nb, mine, group)
        header = frame_header(sizes)
        return ShardedStream(header, sizes, mine, len(header), blob)

    bspec = ErrorSpec(spec.tol, spec.norm, spec.smoothness, Mode.abs)
    if spec.mode == Mode.rel:
        # global normalisation (mgrc.cpp:405-418): tiny all-gather of per-rank stats
        mn, mx, bad, ss = np.inf, -np.inf, 0, 0.0
        for b in mine:
            a, c, nf = block_stats(data[b])
            mn, mx, bad = min(mn, a), max(mx, c), bad | int(nf)
        if spec.norm == Norm.s:
            # Σu² in file order, added serially like the CLI's scan_stats (mgrc.cpp:197-233): with a
            # slowest-axis slab plan every rank holds consecutive rows, so the exact serial sum is a chain
            # (rank r continues from rank r-1's running value; one double passed per rank)
            slabs = all(int(r[1] - r[0]) == shape[a] for blk in plan for a, r in enumerate(blk) if a > 0)
            if slabs:
                ss = _chain_recv(rank, group)
                for b in mine:
                    ss = block_sumsq(data[b], ss)
                _chain_send(ss, rank, world, group)
            else:  # blocks split inner axes: per-rank partials combined in rank order (ulp-level difference)
                for b in mine:
                    ss = ss + block_sumsq(data[b], 0.0)
        st = _allgather_floats([mn, mx, float(bad), ss], group)
        if any(row[2] for row in st):
            raise MgrcError(5, "NonFiniteInput: input contains NaN or Inf")
        gmin = min(row[0] for row in st)
        gmax = max(row[1] for row in st)
        if spec.norm == Norm.inf:
            nrm = gmax - gmin
        else:
            if slabs:  # the last rank holds the whole serial sum
                tot = st[-1][3]
            else:
                tot = 0.0
                for row in st:  # rank order
                    tot = tot + row[3]
            nrm = float(np.sqrt(tot / float(np.prod(shape))))
        if nrm == 0.0:
            raise MgrcError(6, "DegenerateData: relative bound on a constant file")
        bspec = ErrorSpec(spec.tol * nrm, spec.norm, spec.smoothness, Mode.abs)

    cs = [np.arange(s, dtype=np.float64) for s in shape] if coords is None else \
        [np.asarray(c, dtype=np.float64) for c in coords]
    blobs = []
    for b in mine:
        rng = plan[b].tolist()
        bshape = tuple(int(r[1] - r[0]) for r in rng)
        blobs.append(block_compress(data[b], bshape, block_coords(rng, cs), bspec, codec))
    sizes = _allgather_ints([len(x) for x in blobs], nb, mine, group)
    header = frame_header(sizes)
    my_offset = len(header) + sum(sizes[: mine[0]]) if mine else len(header) + sum(sizes)
    return ShardedStream(header, sizes, mine, my_offset, b"".join(blobs))


def decompress_sharded(stream, group=None, block_decompress=None):
    """This rank's slabs of a multiblock stream: [(block, ranges, array)].

    Offsets are validated like ``split_multiblock`` (mgrc.cpp:277-293); no
    collective is needed (each rank reads the offset table).
    """
    import torch.distributed as dist

    from . import decompress, inspect

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    block_decompress = block_decompress or decompress
    buf = bytes(stream)
    if len(buf) < 4:
        raise MgrcError(9, "CorruptStream: truncated stream")
    (count,) = struct.unpack_from("<I", buf, 0)
    if count == 0 or 4 + 8 * count > len(buf):
        raise MgrcError(9, "CorruptStream: bad block table")
    offs = list(struct.unpack_from(f"<{count}Q", buf, 4))
    out = []
    for b in blocks_of(rank, count, world):
        lo = offs[b]
        hi = offs[b + 1] if b + 1 < count else len(buf)
        if lo < 4 + 8 * count or hi > len(buf) or lo > hi:
            raise MgrcError(9, "CorruptStream: bad block offsets")
        blob = buf[lo:hi]
        info = inspect(blob)
        out.append((b, info, block_decompress(blob)))
    return out


def _allgather_ints(local: List[int], nblocks: int, mine: List[int], group) -> List[int]:
    """Per-block sizes in plan order (one small all-gather)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return list(local)
    dev = _coll_device(group)
    vec = torch.zeros(nblocks, dtype=torch.int64, device=dev)
    for b, s in zip(mine, local):
        vec[b] = s
    parts = [torch.zeros_like(vec) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, vec, group=group)
    tot = torch.stack(parts).sum(0)
    return [int(x) for x in tot.cpu().tolist()]


def _allgather_floats(vals: List[float], group) -> List[List[float]]:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [list(vals)]
    dev = _coll_device(group)
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    parts = [torch.zeros_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    return [p.cpu().tolist() for p in parts]


def _chain_recv(rank: int, group) -> float:
    import torch
    import torch.distributed as dist

    if rank == 0 or not dist.is_initialized():
        return 0.0
    t = torch.zeros(1, dtype=torch.float64, device=_coll_device(group))
    dist.recv(t, src=dist.get_global_rank(group, rank - 1) if group is not None else rank - 1, group=group)
    return float(t.item())


def _chain_send(v: float, rank: int, world: int, group) -> None:
    import torch
    import torch.distributed as dist

    if rank + 1 >= world or not dist.is_initialized():
        return
    t = torch.tensor([v], dtype=torch.float64, device=_coll_device(group))
    dist.send(t, dst=dist.get_global_rank(group, rank + 1) if group is not None else rank + 1, group=group)


def _coll_device(group):
    import torch
    import torch.distributed as dist

    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")

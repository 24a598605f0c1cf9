"""Multi-rank host logic of the chunked driver (paper_2401_05994_b200/sharded.py)
on CPU with the ``gloo`` backend, world_size 2 (and 1, 3).

The per-block compressor is injected (the CPU oracle) because this container
has no GPU; the product default is the sm_100a library.  What is checked is
the distributed part: block ownership, the REL all-gather, the all-gather of
sizes, the offset table and the placement — the assembled stream must be
byte-identical to the reference CLI's multiblock stream (oracle
``compress_chunked`` restates tools/mgrc.cpp:363-484) for every world size.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = {
    "inf_rel_f32": dict(shape=(40, 33, 17), dtype="f32", tol=1e-4, norm=0, s=0.0, mode=1, chunk=17 * 33 * 17 * 4),
    "inf_abs_f64_2d": dict(shape=(70, 65), dtype="f64", tol=1e-3, norm=0, s=0.0, mode=0, chunk=20 * 65 * 8),
    "s0_abs_f64": dict(shape=(60, 20, 20), dtype="f64", tol=1e-3, norm=1, s=0.0, mode=0, chunk=17 * 400 * 8),
    "s0_rel_f64": dict(shape=(60, 20, 20), dtype="f64", tol=1e-3, norm=1, s=0.0, mode=1, chunk=17 * 400 * 8),
    "s1_rel_f32": dict(shape=(50, 24, 20), dtype="f32", tol=1e-3, norm=1, s=1.0, mode=1, chunk=17 * 24 * 20 * 4),
    "single_block": dict(shape=(33, 17), dtype="f64", tol=1e-3, norm=0, s=0.0, mode=1, chunk=0),
}


def _worker(rank, world, port, case_name, out_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2401_05994_b200 as mg
        from paper_2401_05994_b200 import sharded
        from oracle import binding

        orc = binding.get("restatement")
        c = CASES[case_name]
        u = orc.multisine_noisy(c["shape"], 42, 0.05).astype(np.float32 if c["dtype"] == "f32" else np.float64)

        def read_block(b, ranges):
            sl = tuple(slice(int(r[0]), int(r[1])) for r in ranges)
            return np.ascontiguousarray(u[sl])

        def block_compress(block, bshape, coords, spec, codec):
            return orc.compress(block, spec.tol, int(spec.norm), spec.smoothness, int(spec.mode), int(codec),
                                coords=coords, shape=bshape)

        def block_sumsq(block, s0):  # the CLI's serial accumulation (mgrc.cpp:227), continued from s0
            acc = float(s0)
            for v in np.asarray(block, dtype=np.float64).ravel().tolist():
                acc = acc + v * v
            return acc

        def block_stats(block):
            b = np.asarray(block, dtype=np.float64)
            return float(b.min()), float(b.max()), bool(~np.isfinite(b).all())

        spec = mg.ErrorSpec(c["tol"], mg.Norm(c["norm"]), c["s"], mg.Mode(c["mode"]))
        st = sharded.compress_sharded(read_block, c["shape"], mg.DType.f32 if c["dtype"] == "f32" else mg.DType.f64,
                                      spec, mg.Codec.huffman, chunk_mem=c["chunk"], block_compress=block_compress,
                                      block_stats=block_stats, block_sumsq=block_sumsq)
        # assemble on every rank through an all-gather of the parts (test only)
        parts = [None] * world
        dist.all_gather_object(parts, (st.my_offset, st.my_bytes))
        buf = bytearray(st.total_len)
        buf[: len(st.header)] = st.header
        for off, by in parts:
            buf[off: off + len(by)] = by
        # decompress: each rank its own slabs, no collective
        dec = sharded.decompress_sharded(bytes(buf), block_decompress=orc.decompress)
        out_q.put((rank, bytes(buf), [(b, arr.shape) for b, _, arr in dec]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("case_name", sorted(CASES))
def test_sharded_stream_matches_cli(case_name, world):
    from oracle import binding

    orc = binding.get("restatement")
    c = CASES[case_name]
    u = orc.multisine_noisy(c["shape"], 42, 0.05).astype(np.float32 if c["dtype"] == "f32" else np.float64)
    want = orc.compress_chunked(u, c["tol"], c["norm"], c["s"], c["mode"], 2, chunk_mem=c["chunk"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    blocks_seen = []
    for rank, stream, dec in res:
        assert stream == want, (rank, world)  # S-REL too: the serial Σu² is chained rank to rank
        blocks_seen += [b for b, _ in dec]
    nb = int.from_bytes(want[:4], "little")
    assert sorted(blocks_seen) == list(range(nb))


def test_ownership_contiguous():
    from paper_2401_05994_b200 import sharded

    for nb in (1, 3, 8, 9, 16):
        for world in (1, 2, 4, 8):
            owners = [sharded.owner_of(b, nb, world) for b in range(nb)]
            assert owners == sorted(owners)
            assert set(owners) <= set(range(world))
    assert [sharded.owner_of(b, 8, 8) for b in range(8)] == list(range(8))

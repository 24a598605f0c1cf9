"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle.

Bar (north_star / SURVEY §8): containers byte-identical to the reference's
(which implies bit-exact quantised codes, identical Huffman bytes and an
identical ratio), decompressed arrays bit-identical to the reference's
decompressor, and every reconstruction within the requested bound.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# (shape, dtype, tol, norm, s, mode, field)
CASES = [
    ((65, 65, 65), np.float64, 1e-3, 0, 0.0, 1, "multisine"),        # config 1
    ((33, 17, 9), np.float32, 1e-4, 0, 0.0, 1, "noisy"),
    ((129, 130), np.float64, 1e-3, 1, 1.0, 1, "noisy"),             # S(1), level-weighted estimator
    ((129, 130), np.float64, 1e-3, 1, 0.0, 1, "noisy"),             # S(0) = RMS
    ((257, 256), np.float32, 1e-5, 0, 0.0, 1, "noisy"),
    ((12, 7, 10), np.float32, 1e-3, 1, 0.0, 0, "noisy"),
    ((6, 5, 4, 3), np.float64, 1e-2, 0, 0.0, 0, "noisy"),           # 4-D
    ((17,), np.float64, 1e-3, 0, 0.0, 1, "noisy"),                  # 1-D
    ((6,), np.float64, 1e-3, 0, 0.0, 0, "noisy"),
    ((2, 2), np.float64, 1e-3, 0, 0.0, 0, "noisy"),                 # L = 0
    ((2, 9), np.float32, 1e-3, 0, 0.0, 0, "noisy"),
    ((256, 33), np.float32, 1e-4, 1, 0.0, 1, "noisy"),              # f32 S(0): cast-error RMS
    ((100, 3, 40), np.float64, 1e-6, 0, 0.0, 0, "random"),         # wide codes
    ((65, 65), np.float64, 1e-14, 0, 0.0, 0, "random"),            # |q| > 2^31 (u64 path)
]


def field(oracle, kind, shape, dtype):
    if kind == "multisine":
        u = oracle.multisine(shape)
    elif kind == "noisy":
        u = oracle.multisine_noisy(shape, 42, 0.05)
    else:
        u = oracle.random_field(shape, 7, -3.0, 3.0)
    return u.astype(dtype)


@pytest.mark.parametrize("codec", [2, 1, 0])
@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[0])) + f"-{c[1].__name__}-n{c[3]}s{c[4]}")
def test_container_parity(mg, oracle, case, codec):
    shape, dt, tol, norm, s, mode, kind = case
    u = field(oracle, kind, shape, dt)
    want = oracle.compress(u, tol, norm, s, mode, codec)
    got = mg.compress(u, mg.make_grid(shape), mg.ErrorSpec(tol, mg.Norm(norm), s, mg.Mode(mode)), mg.Codec(codec))
    assert len(got) == len(want)
    assert got == want
    # decompress on the GPU == reference decompressor, bit for bit
    back = mg.decompress(got)
    ref_back = oracle.decompress(want)
    assert back.dtype == ref_back.dtype and back.shape == ref_back.shape
    assert np.array_equal(back.view(np.uint8), ref_back.view(np.uint8))


def test_decompress_accepts_device_buffers(mg, oracle):
    import torch

    u = field(oracle, "noisy", (33, 40, 21), np.float32)
    blob = oracle.compress(u, 1e-4, 0, 0.0, 1, 2)
    dblob = torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda()
    out = torch.empty(u.shape, dtype=torch.float32, device="cuda")
    mg.decompress_into(dblob, out)
    assert np.array_equal(out.cpu().numpy(), oracle.decompress(blob))
    # compress from a device tensor into a device buffer
    du = torch.from_numpy(u).cuda()
    n = mg.compress_to(du, None, mg.make_grid(u.shape), mg.ErrorSpec(1e-4, mg.Norm.inf, 0.0, mg.Mode.rel))
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda")
    mg.compress_to(du, dst, mg.make_grid(u.shape), mg.ErrorSpec(1e-4, mg.Norm.inf, 0.0, mg.Mode.rel))
    assert bytes(dst.cpu().numpy()) == blob


def test_explicit_coords(mg, oracle):
    rng = np.random.default_rng(3)
    shape = (17, 12, 9)
    coords = [np.cumsum(rng.uniform(0.05, 1.0, n)) - 1.0 for n in shape]
    u = field(oracle, "noisy", shape, np.float64)
    want = oracle.compress(u, 1e-3, 0, 0.0, 0, 2, coords=coords)
    got = mg.compress(u, mg.make_grid(shape, coords), mg.ErrorSpec(1e-3))
    assert got == want
    assert np.array_equal(mg.decompress(got), oracle.decompress(want))


@pytest.mark.parametrize("value", [3.25, 0.0, -0.0])
def test_constant_field(mg, oracle, value):
    u = np.full((9, 33), value)
    want = oracle.compress(u, 1e-3, 0, 0.0, 1, 2)
    got = mg.compress(u, mg.make_grid(u.shape), mg.ErrorSpec(1e-3, mg.Norm.inf, 0.0, mg.Mode.rel))
    assert got == want
    assert np.array_equal(mg.decompress(got).view(np.uint64), oracle.decompress(want).view(np.uint64))


def test_error_paths(mg, oracle):
    u = field(oracle, "noisy", (9, 17), np.float64)
    grid = mg.make_grid(u.shape)
    bad = u.copy()
    bad[3, 3] = np.nan
    with pytest.raises(mg.MgrcError) as e:
        mg.compress(bad, grid, mg.ErrorSpec(1e-3))
    assert e.value.name == "NonFiniteInput"
    with pytest.raises(mg.MgrcError) as e:
        mg.compress(u, grid, mg.ErrorSpec(0.0))
    assert e.value.name == "InvalidState"
    with pytest.raises(mg.MgrcError) as e:
        mg.compress(u, mg.make_grid((9, 1)), mg.ErrorSpec(1e-3))
    assert e.value.name == "InvalidShape"
    with pytest.raises(mg.MgrcError) as e:
        mg.compress(u, grid, mg.ErrorSpec(1e-300, mg.Norm.inf))
    assert e.value.name == "Overflow"
    blob = oracle.compress(u, 1e-3, 0, 0.0, 0, 2)
    flipped = bytearray(blob)
    flipped[-5] ^= 0x10
    with pytest.raises(mg.MgrcError) as e:
        mg.decompress(bytes(flipped))
    assert e.value.name == "ChecksumMismatch"
    with pytest.raises(mg.MgrcError) as e:
        mg.decompress(blob[:-1])
    assert e.value.name == "CorruptStream"


def test_corrupt_streams_match_reference_errors(mg, oracle):
    """Byte-flip fuzzing of codec-2 payloads with the CRC recomputed, so the
    decoder itself must detect the damage exactly where the reference does."""
    import zlib

    u = field(oracle, "noisy", (33, 20), np.float64)
    blob = bytearray(oracle.compress(u, 1e-3, 0, 0.0, 0, 2))
    info = oracle.inspect(bytes(blob))
    hs, pl = info.header_size, info.payload_len
    rng = np.random.default_rng(11)
    for trial in range(60):
        b = bytearray(blob)
        k = int(rng.integers(3 + 128, pl))  # inside the code stream
        b[hs + k] ^= int(rng.integers(1, 256))
        crc = zlib.crc32(bytes(b[hs:hs + pl]))
        b[hs - 4:hs] = crc.to_bytes(4, "little")
        b = bytes(b)
        try:
            want = oracle.decompress(b)
            werr = None
        except Exception as e:  # noqa: BLE001
            werr = e.name
        try:
            got = mg.decompress(b)
            gerr = None
        except mg.MgrcError as e:
            gerr = e.name
        assert gerr == werr, (trial, gerr, werr)
        if werr is None:
            assert np.array_equal(got, want)


# ---------------------------------------------------------------------------
# BASELINE.json configurations at full size: the container the
# GPU produces is byte-identical to the CPU reference's on the same input
# bytes, and the GPU decompressor reproduces the reference decompressor's
# output bit for bit.  (cfg 2: ~30 s of CPU oracle time; cfg 3: ~15 s.)
FULL = [
    ("cfg2_513cubed_f32_inf_rel1e-4", (513, 513, 513), np.float32, 1e-4, 0, 0.0, 1),
    ("cfg3_8193sq_f64_s1_rel1e-3", (8193, 8193), np.float64, 1e-3, 1, 1.0, 1),
]


@pytest.mark.slow
@pytest.mark.parametrize("case", FULL, ids=lambda c: c[0])
def test_full_size_parity(mg, oracle, case):
    name, shape, dt, tol, norm, s, mode = case
    u = oracle.multisine(shape).astype(dt)
    spec = mg.ErrorSpec(tol, mg.Norm(norm), s, mg.Mode(mode))
    got = mg.compress(u, mg.make_grid(shape), spec, mg.Codec.huffman)
    from oracle import binding

    if binding.available("reference"):  # the reference library itself (OpenMP), else the restatement
        oracle = binding.get("reference")
        oracle.set_threads(os.cpu_count() or 1)
    want = oracle.compress(u, tol, norm, s, mode, 2)
    assert len(got) == len(want)
    assert got == want
    back = mg.decompress(want)
    ref_back = oracle.decompress(want)
    assert np.array_equal(back.view(np.uint8), ref_back.view(np.uint8))
    if norm == 0:
        tau = tol * float(u.max() - u.min())
        assert float(np.max(np.abs(back.astype(np.float64) - u))) <= tau


# ---------------------------------------------------------------------------
# Chunked (multiblock) streams: the C-ABI's one-GPU CLI driver and the
# multi-rank driver (world size 1 here; the collective logic is covered by the
# gloo tests) against the restated CLI (tools/mgrc.cpp:363-542).
CHUNKED = [
    ((40, 33, 17), np.float32, 1e-4, 0, 0.0, 1, 17 * 33 * 17 * 4),
    ((70, 65), np.float64, 1e-3, 0, 0.0, 0, 20 * 65 * 8),
    ((60, 20, 20), np.float64, 1e-3, 1, 0.0, 1, 17 * 400 * 8),   # S-REL: the CLI's serial Σu² order
]


@pytest.mark.parametrize("case", CHUNKED, ids=lambda c: "x".join(map(str, c[0])))
def test_chunked_parity(mg, oracle, case):
    shape, dt, tol, norm, s, mode, cm = case
    u = oracle.multisine_noisy(shape, 42, 0.05).astype(dt)
    want = oracle.compress_chunked(u, tol, norm, s, mode, 2, chunk_mem=cm)
    got = mg.compress_chunked(u, mg.ErrorSpec(tol, mg.Norm(norm), s, mg.Mode(mode)), mg.Codec.huffman, chunk_mem=cm)
    assert got == want
    assert np.array_equal(mg.decompress_chunked(got), oracle_decompress_chunked(oracle, want, shape))
    from paper_2401_05994_b200 import sharded  # the multi-rank driver (world size 1 here), S-REL included

    def read_block(b, ranges):
        return np.ascontiguousarray(u[tuple(slice(int(r[0]), int(r[1])) for r in ranges)])

    st = sharded.compress_sharded(read_block, shape, mg.DType.f32 if dt == np.float32 else mg.DType.f64,
                                  mg.ErrorSpec(tol, mg.Norm(norm), s, mg.Mode(mode)), mg.Codec.huffman, chunk_mem=cm)
    buf = bytearray(st.total_len)
    st.write_into(buf)
    assert bytes(buf) == want


def test_serial_sumsq_matches_cli_scan(mg, oracle):
    """The CLI's scan_stats accumulation (mgrc.cpp:227: sumsq += v*v in file order), bit-exact, host and device
    arrays, and continued across a split (the multi-rank chain)."""
    import torch

    for dt in (np.float32, np.float64):
        u = oracle.multisine_noisy((37, 41, 13), 42, 0.05).astype(dt)
        want = 0.0
        for v in u.astype(np.float64).ravel().tolist():
            want = want + v * v
        assert mg.serial_sumsq(u) == want
        assert mg.serial_sumsq(torch.from_numpy(u).cuda()) == want
        a = mg.serial_sumsq(np.ascontiguousarray(u[:20]))
        assert mg.serial_sumsq(np.ascontiguousarray(u[20:]), a) == want


def oracle_decompress_chunked(oracle, stream, shape):
    """Reassemble the reference decompressor's per-block output (tools/mgrc.cpp:490-542)."""
    import struct

    count = struct.unpack_from("<I", stream, 0)[0]
    offs = list(struct.unpack_from(f"<{count}Q", stream, 4)) + [len(stream)]
    parts = [oracle.decompress(stream[offs[i]:offs[i + 1]]) for i in range(count)]
    return np.concatenate(parts, axis=0).reshape(shape)


# ---------------------------------------------------------------------------
# configs[3] (1025^3 f64, INF REL 1e-5) and configs[4] (2049^3 f32 slabs): the
# full sizes are checked through size-independent properties (bound met,
# deterministic containers, decompress(compress(u)) reproducible); byte parity
# with the reference is checked on sub-fields of the same generator and
# tolerance (257^3 f64 at 1e-5; a 65 x 2049 x 2049 f32 slab of the 2049^3
# field, whose stream exercises the long-desynchronisation decode path).
@pytest.mark.slow
def test_cfg4_subfield_parity(mg, oracle):
    u = oracle.multisine((257, 257, 257))
    from oracle import binding

    ref = binding.get("reference") if binding.available("reference") else oracle
    ref.set_threads(os.cpu_count() or 1)
    want = ref.compress(u, 1e-5, 0, 0.0, 1, 2)
    got = mg.compress(u, mg.make_grid(u.shape), mg.ErrorSpec(1e-5, mg.Norm.inf, 0.0, mg.Mode.rel))
    assert got == want
    assert np.array_equal(mg.decompress(got), ref.decompress(want))


@pytest.mark.slow
def test_cfg4_full_size_properties(mg):
    import torch

    from bench import multisine_torch

    u = multisine_torch((1025, 1025, 1025), "cuda")
    spec = mg.ErrorSpec(1e-5, mg.Norm.inf, 0.0, mg.Mode.rel)
    grid = mg.make_grid(u.shape)
    n1 = mg.compress_to(u, None, grid, spec)
    dst = torch.empty(n1, dtype=torch.uint8, device="cuda")
    assert mg.compress_to(u, dst, grid, spec) == n1
    dst2 = torch.empty(n1, dtype=torch.uint8, device="cuda")
    mg.compress_to(u, dst2, grid, spec)
    assert torch.equal(dst, dst2)  # deterministic container
    out = torch.empty_like(u)
    mg.decompress_into(dst, out)
    tau = 1e-5 * float(u.max() - u.min())
    assert float((out - u).abs().max()) <= tau
    out2 = torch.empty_like(u)
    mg.decompress_into(dst, out2)
    assert torch.equal(out, out2)


@pytest.mark.slow
def test_cfg5_slab_parity(mg, oracle):
    import torch

    from bench import multisine_rows

    shape = (2049, 2049, 2049)
    u = multisine_rows(shape, 0, 65, "cuda").to(torch.float32).contiguous().cpu().numpy()
    tau = 1e-4 * 4.0  # an ABS bound of the order of the global REL one
    from oracle import binding

    ref = binding.get("reference") if binding.available("reference") else oracle
    ref.set_threads(os.cpu_count() or 1)
    want = ref.compress(u, tau, 0, 0.0, 0, 2)
    got = mg.compress(u, mg.make_grid(u.shape), mg.ErrorSpec(tau, mg.Norm.inf, 0.0, mg.Mode.abs))
    assert got == want
    back = mg.decompress(want)
    assert np.array_equal(back, ref.decompress(want))

"""GPU parity, round 2: the cases round 1 never compared on the device.

* every golden container the REFERENCE produced (tests/golden/, which includes
  65^3 S(0) REL 1e-3 and the constant / coords / codec 0-1 cases) is
  reproduced byte for byte by the sm_100a path, and the GPU decompressor
  reproduces the reference decompressor's output digest;
* f32 data at tolerances near the f32 cast error (container.cpp:96-110) —
  where the a-priori bound cannot decide, the exact a-posteriori check with
  the cast epilogue runs, the shrink loop takes >= 2 passes, and at 1e-8 the
  reference gives up with ToleranceUnreachable (container.cpp:118-121);
* skewed 2-D streams whose natural Huffman depth exceeds 15 bits, so the
  Kraft repair of build_lengths (codec.cpp:157-190) shapes the table
  (2049^2 INF REL 1e-3: depth 16; 8193^2 S(0) REL 1e-3: depth 17);
* BASELINE configs[3] (1025^3 f64 INF REL 1e-5) at full size, and configs[4]
  (2049^3 f32, the CLI's 8-slab plan with chunk_mem 4,315,956,228 and the
  global REL bound) slab by slab, against the reference library.
"""
import hashlib
import json
import os
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"
MAN = json.loads((GOLD / "manifest.json").read_text())


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def make_field(o, kind, shape, dtype):
    if kind == "multisine":
        u = o.multisine(shape)
    elif kind == "noisy":
        u = o.multisine_noisy(shape, 42, 0.05)
    elif kind == "random":
        u = o.random_field(shape, 7, -3.0, 3.0)
    elif kind.startswith("const"):
        u = np.full(shape, float(kind[5:]))
    else:
        raise ValueError(kind)
    return u.astype(np.float32 if dtype == "f32" else np.float64)


def make_coords(shape, seed):
    rng = np.random.default_rng(seed)
    return [np.cumsum(rng.uniform(0.05, 1.0, n)) - 1.0 for n in shape]


def reference(oracle):
    """The compiled reference library when present (OpenMP, all host threads), else the restatement."""
    from oracle import binding

    r = binding.get("reference") if binding.available("reference") else oracle
    r.set_threads(os.cpu_count() or 1)
    return r


@pytest.mark.parametrize("case", MAN["containers"], ids=lambda c: c["name"])
def test_golden_containers_on_gpu(mg, oracle, case):
    u = make_field(oracle, case["field"], tuple(case["shape"]), case["dtype"])
    assert sha(u) == case["input_sha256"]
    coords = make_coords(case["shape"], case["coords_seed"]) if case["coords_seed"] is not None else None
    spec = mg.ErrorSpec(case["tol"], mg.Norm(case["norm"]), case["s"], mg.Mode(case["mode"]))
    got = mg.compress(u, mg.make_grid(u.shape, coords), spec, mg.Codec(case["codec"]))
    gold = (GOLD / f"{case['name']}.mgrc").read_bytes()
    assert len(got) == case["container_len"]
    assert got == gold
    assert sha(mg.decompress(gold)) == case["output_sha256"]
    assert mg.describe(gold) == case["describe"]


@pytest.mark.parametrize("case", MAN["chunked"], ids=lambda c: c["name"])
def test_golden_chunked_on_gpu(mg, oracle, case):
    u = make_field(oracle, case["field"], tuple(case["shape"]), case["dtype"])
    spec = mg.ErrorSpec(case["tol"], mg.Norm(case["norm"]), case["s"], mg.Mode(case["mode"]))
    got = mg.compress_chunked(u, spec, mg.Codec.huffman, chunk_mem=case["chunk_mem"])
    assert got == (GOLD / f"{case['name']}.mgrcm").read_bytes()


# ---------------------------------------------------------------------------
# the exact a-posteriori check, shrink passes and ToleranceUnreachable


TIGHT = [  # (dtype, shape, field, tol, norm, mode) — the f64 cases need 2-4 shrink passes in the reference
    ("f64", (17,), "multisine", 5.62341325190349e-17, 0, 0),
    ("f64", (65,), "multisine", 1.1231045018329515e-16, 0, 0),
    ("f64", (9, 9), "random", 4.523370744772097e-16, 0, 0),
    ("f64", (33, 17), "noisy", 5.596276445319564e-17, 1, 0),    # S(0)
    ("f32", (33, 17, 9), "multisine", 1e-7, 0, 1),             # f32 cast check near the f32 ulp
    ("f32", (33, 17, 9), "multisine", 1e-8, 0, 1),
    ("f32", (65, 40), "noisy", 2e-8, 0, 1),
    ("f32", (40, 33, 17), "noisy", 1e-8, 1, 1),                # S(0), f32 cast-error RMS
    ("f32", (9, 8, 7, 6), "noisy", 1e-7, 0, 1),                # 4-D
    ("f32", (2, 3), "noisy", 1e-7, 0, 1),                      # L = 0
]


def _try(fn):
    try:
        return fn(), None
    except Exception as e:  # noqa: BLE001 - both sides raise their own error type with .name
        return None, getattr(e, "name", type(e).__name__)


def _passes(info, tau, d, norm):
    """Shrink passes the reference ran: log2(initial / final bin width) + 1 (error_control.cpp:42-60)."""
    import math

    L = info.nlevels
    w0 = 2 * tau / (1 + L * 2 ** d) if norm == 0 else 2 * tau / math.sqrt((L + 1) * 2 ** d)
    return round(math.log2(w0 / info.bin_widths[0])) + 1


def _match(mg, oracle, dt, shape, kind, tol, norm, mode):
    u = make_field(oracle, kind, shape, dt)
    want, werr = _try(lambda: oracle.compress(u, tol, norm, 0.0, mode, 2))
    spec = mg.ErrorSpec(tol, mg.Norm(norm), 0.0, mg.Mode(mode))
    got, gerr = _try(lambda: mg.compress(u, mg.make_grid(shape), spec, mg.Codec.huffman))
    assert gerr == werr, (shape, tol, gerr, werr)
    if werr is not None:
        return None
    assert got == want, (shape, tol)
    st = mg.last_compress_stats()
    back = mg.decompress(got)
    assert np.array_equal(back, oracle.decompress(want))
    err = back.astype(np.float64) - u.astype(np.float64)
    if st["decided_by"] != "none" and dt == "f32":  # f32 data: the reference checks the cast-back output
        measured = np.max(np.abs(err)) if norm == 0 else np.sqrt(np.mean(err * err))
        assert measured <= st["tau_abs"]
    info = mg.inspect(got)
    if info.nlevels >= 1 and mode == 0:
        assert st["passes"] == _passes(info, tol, len(shape), norm), (shape, tol)
    return st


def test_tight_tolerances_match_reference(mg, oracle):
    """Byte parity where the shrink loop (container.cpp:93-123) runs more than one pass and the exact
    a-posteriori check decides; the pass count equals the reference's (from its final bin widths)."""
    passes = []
    for case in TIGHT:
        st = _match(mg, oracle, *case)
        if st:
            passes.append(st["passes"])
    assert max(passes) >= 3, passes


def test_rounding_edge_sweep_matches_reference(mg, oracle):
    """ABS tolerances from 1e-14 down to where |c/delta| >= 2^63 (Overflow): every container, pass count
    and error code equals the reference's.  (ToleranceUnreachable needs 10 failed passes, but the codes
    overflow first on every field tried: the reference's own loop cannot reach it at these sizes.)"""
    errs = set()
    for tol in np.geomspace(1e-14, 1e-18, 25):
        for dt, shape, kind, norm in [("f64", (65,), "multisine", 0), ("f64", (9, 9), "random", 0),
                                      ("f64", (33, 17), "noisy", 1), ("f32", (17, 9), "noisy", 0)]:
            if _match(mg, oracle, dt, shape, kind, float(tol), norm, 0) is None:
                errs.add("err")
    assert errs  # the sweep reaches the Overflow edge


def test_exact_check_path_is_taken(mg, oracle):
    """Where rounding makes max|r| exceed delta/2 the a-priori bound cannot decide: the exact a-posteriori
    check runs (and here the loop shrinks twice); at an ordinary tolerance the bound decides."""
    u = make_field(oracle, "multisine", (65,), "f64")
    mg.compress(u, mg.make_grid(u.shape), mg.ErrorSpec(1.1231045018329515e-16, mg.Norm.inf, 0.0, mg.Mode.abs))
    st = mg.last_compress_stats()
    assert st["decided_by"] == "exact" and st["passes"] == 2
    mg.compress(u, mg.make_grid(u.shape), mg.ErrorSpec(1e-4, mg.Norm.inf, 0.0, mg.Mode.rel))
    assert mg.last_compress_stats()["decided_by"] == "bound"


# ---------------------------------------------------------------------------
# Kraft repair on real containers


def _max_code_len(blob, info):
    tab = blob[info.header_size + 3: info.header_size + 3 + 128]
    lens = [b & 15 for b in tab] + [b >> 4 for b in tab]
    return max(lens), blob[info.header_size + 2]


@pytest.mark.slow
@pytest.mark.parametrize("case", [
    ("2049sq_f64_inf_rel1e-3", (2049, 2049), 1e-3, 0, 0.0),
    ("8193sq_f64_s0_rel1e-3", (8193, 8193), 1e-3, 1, 0.0),
], ids=lambda c: c[0])
def test_kraft_repair_full_size(mg, oracle, case):
    _, shape, tol, norm, s = case
    u = oracle.multisine(shape)
    spec = mg.ErrorSpec(tol, mg.Norm(norm), s, mg.Mode.rel)
    got = mg.compress(u, mg.make_grid(shape), spec, mg.Codec.huffman)
    ref = reference(oracle)
    want = ref.compress(u, tol, norm, s, 1, 2)
    assert len(got) == len(want)
    assert got == want
    info = mg.inspect(got)
    maxlen, hdr_maxlen = _max_code_len(got, info)
    assert maxlen == 15 and hdr_maxlen == 15  # clamped: the natural depth is 16 / 17
    back = mg.decompress(got)
    assert np.array_equal(back.view(np.uint64), ref.decompress(want).view(np.uint64))


# ---------------------------------------------------------------------------
# BASELINE configs[3] and configs[4] at full size


@pytest.mark.slow
def test_cfg4_full_size_parity(mg, oracle):
    """1025^3 f64 INF REL 1e-5: the GPU container is byte-identical to the reference library's and the GPU
    decompressor reproduces the reference decompressor bit for bit (the reference needs ~52 GB of RAM)."""
    shape = (1025, 1025, 1025)
    u = oracle.multisine(shape)
    spec = mg.ErrorSpec(1e-5, mg.Norm.inf, 0.0, mg.Mode.rel)
    got = mg.compress(u, mg.make_grid(shape), spec, mg.Codec.huffman)
    ref = reference(oracle)
    want = ref.compress(u, 1e-5, 0, 0.0, 1, 2)
    assert len(got) == len(want)
    assert got == want
    del want
    back = mg.decompress(got)
    tau = 1e-5 * float(u.max() - u.min())
    assert float(np.max(np.abs(back - u))) <= tau
    ref_back = ref.decompress(got)
    assert np.array_equal(back.view(np.uint64), ref_back.view(np.uint64))


CFG5_CHUNK_MEM = 257 * 2049 * 2049 * 4


@pytest.mark.slow
def test_cfg5_slabs_parity(mg, oracle):
    """2049^3 f32, INF REL 1e-4, chunk_mem 4,315,956,228 -> 8 slabs [257, 256x7] (tools/mgrc.cpp:363-484).

    The GPU's multiblock stream (global REL range over the whole field, per-slab ABS containers with the
    slab's index coordinates) is compared slab by slab with the reference library compressing the same slab
    bytes under the same global tau.  By default slabs 0 (257 rows) and 7 (the last) are checked; set
    MGRC_CFG5_ALL_SLABS=1 to check all eight (about 10 minutes of host CPU)."""
    import struct

    import torch

    from bench import multisine_rows

    shape = (2049, 2049, 2049)
    plan = mg.plan_chunks(shape, mg.DType.f32, CFG5_CHUNK_MEM)
    assert [int(r[0][1] - r[0][0]) for r in plan] == [257] + [256] * 7
    u = torch.empty(shape, dtype=torch.float32, device="cuda")
    for a in range(0, shape[0], 64):
        b = min(shape[0], a + 64)
        u[a:b] = multisine_rows(shape, a, b, "cuda").to(torch.float32)
    mn, mx = float(u.min()), float(u.max())
    tau = 1e-4 * (float(np.float64(mx)) - float(np.float64(mn)))
    # the C-ABI's one-GPU CLI driver on the device-resident field
    spec = mg.ErrorSpec(1e-4, mg.Norm.inf, 0.0, mg.Mode.rel)
    stream = mg.compress_chunked(u, spec, mg.Codec.huffman, chunk_mem=CFG5_CHUNK_MEM)
    count = struct.unpack_from("<I", stream, 0)[0]
    assert count == 8
    offs = list(struct.unpack_from("<8Q", stream, 4)) + [len(stream)]
    assert offs[0] == 4 + 8 * 8
    slabs = range(8) if os.environ.get("MGRC_CFG5_ALL_SLABS") else (0, 7)
    ref = reference(oracle)
    for b in slabs:
        r0, r1 = int(plan[b][0][0]), int(plan[b][0][1])
        slab = u[r0:r1].cpu().numpy()
        coords = [np.arange(r0, r1, dtype=np.float64), np.arange(2049, dtype=np.float64),
                  np.arange(2049, dtype=np.float64)]
        want = ref.compress(slab, tau, 0, 0.0, 0, 2, coords=coords)
        blk = stream[offs[b]:offs[b + 1]]
        assert len(blk) == len(want), b
        assert blk == want, b
        back = mg.decompress(blk)
        assert np.array_equal(back, ref.decompress(want)), b
        assert float(np.max(np.abs(back.astype(np.float64) - slab.astype(np.float64)))) <= tau
        del slab, want, back


# ---------------------------------------------------------------------------
# S(s != 0): the accept decision is certified against the reference's serial
# per-level sums (error_control.cpp:72-101); the exact serial fallback is
# forced here (MGRC_LW_CERTIFY=serial) and must give the same containers.


@pytest.mark.parametrize("case", [
    ((129, 130), "noisy", 1e-3, 1.0),
    ((65, 33, 17), "noisy", 1e-3, 1.0),
    ((257, 256), "multisine", 1e-4, 0.5),
    ((33, 9, 8, 5), "noisy", 1e-2, 2.0),
], ids=lambda c: "x".join(map(str, c[0])) + f"-s{c[3]}")
def test_level_weighted_serial_fallback(mg, oracle, case, monkeypatch):
    shape, kind, tol, s = case
    u = make_field(oracle, kind, shape, "f64")
    want = oracle.compress(u, tol, 1, s, 1, 2)
    spec = mg.ErrorSpec(tol, mg.Norm.s, s, mg.Mode.rel)
    got = mg.compress(u, mg.make_grid(shape), spec, mg.Codec.huffman)
    assert got == want
    fast = mg.last_compress_stats()
    assert fast["decided_by"] == "exact"
    monkeypatch.setenv("MGRC_LW_CERTIFY", "serial")
    got2 = mg.compress(u, mg.make_grid(shape), spec, mg.Codec.huffman)
    st = mg.last_compress_stats()
    assert st["decided_by"] == "exact-serial"
    assert got2 == want
    # the exact fallback reproduces the reference's estimator bit for bit (one pass: final widths = initial)
    _, r, _ = oracle.quantize(oracle.forward(u), mg.inspect(want).bin_widths)
    assert st["achieved"] == oracle.achieved_error(r, 1, s)
    # the tree estimate is within the certified window of the serial value
    assert abs(fast["achieved"] - st["achieved"]) <= 1e-12 * st["achieved"]


# ---------------------------------------------------------------------------
# the single-process multi-GPU chunked driver (mgrc_gpu_compress_chunked_multi):
# the stream is byte-identical for every rank count (ranks share the device on
# a one-GPU box; the NCCL all-gather runs when they sit on distinct devices)


@pytest.mark.parametrize("case", [
    ((40, 33, 17), "multisine", "f32", 1e-4, 0, 0.0, 1, 17 * 33 * 17 * 4),
    ((70, 65), "noisy", "f64", 1e-3, 0, 0.0, 0, 20 * 65 * 8),
    ((60, 20, 20), "noisy", "f64", 1e-3, 1, 0.0, 1, 17 * 400 * 8),   # S-REL: the serial Σu² order
    ((100, 70), "noisy", "f64", 1e-3, 0, 0.0, 1, 17 * 70 * 8),
], ids=lambda c: "x".join(map(str, c[0])))
@pytest.mark.parametrize("ngpus", [2, 3, 8])
def test_chunked_multi_rank(mg, oracle, case, ngpus):
    shape, kind, dt, tol, norm, s, mode, cm = case
    u = make_field(oracle, kind, shape, dt)
    spec = mg.ErrorSpec(tol, mg.Norm(norm), s, mg.Mode(mode))
    want = oracle.compress_chunked(u, tol, norm, s, mode, 2, chunk_mem=cm)
    got = mg.compress_chunked(u, spec, mg.Codec.huffman, chunk_mem=cm, ngpus=ngpus)
    assert got == want
    assert np.array_equal(mg.decompress_chunked(got, ngpus=ngpus), mg.decompress_chunked(got))


# ---------------------------------------------------------------------------
# device-resident containers at every body alignment (the library copies the
# body into its padded, aligned buffer): the host path's output and errors


@pytest.mark.parametrize("case", [((65, 33, 17), "noisy", "f32", 1e-4), ((129, 130), "random", "f64", 1e-3),
                                  ((33, 9, 8, 5), "noisy", "f64", 1e-2)], ids=lambda c: "x".join(map(str, c[0])))
def test_device_containers_in_place_and_copied(mg, oracle, case):
    import torch

    shape, kind, dt, tol = case
    u = make_field(oracle, kind, shape, dt)
    blob = mg.compress(u, mg.make_grid(shape), mg.ErrorSpec(tol, mg.Norm.inf, 0.0, mg.Mode.rel))
    want = mg.decompress(blob)
    raw = torch.frombuffer(bytearray(blob), dtype=torch.uint8)
    for shift in range(4):  # the body's alignment cycles through 0..3 bytes
        buf = torch.zeros(len(blob) + shift + 256, dtype=torch.uint8, device="cuda")
        dev = buf[shift:shift + len(blob)]
        dev.copy_(raw.cuda())
        out = torch.empty(shape, dtype=torch.float32 if dt == "f32" else torch.float64, device="cuda")
        mg.decompress_into(dev, out)
        assert np.array_equal(out.cpu().numpy(), want)
        # a flipped bit in the body: the same error as the host path
        bad = bytearray(blob)
        bad[len(bad) - 20] ^= 0x10
        try:
            mg.decompress(bytes(bad))
            host_err = None
        except mg.MgrcError as e:
            host_err = e.name
        dev.copy_(torch.frombuffer(bad, dtype=torch.uint8).cuda())
        try:
            mg.decompress_into(dev, out)
            dev_err = None
        except mg.MgrcError as e:
            dev_err = e.name
        assert dev_err == host_err

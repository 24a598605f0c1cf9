"""The command-line tool (integration/mgrc_cli.cpp):
tools/mgrc.cpp's compress / decompress / inspect over the C-ABI.

CPU tests: argument handling, the raw-file size check and ``inspect`` (header
only) against the oracle's ``describe`` of each block of an oracle-made
multiblock file.  GPU tests: the files the tool writes are byte-identical to
the reference CLI's multiblock compress (oracle ``compress_chunked`` restates
mgrc.cpp:363-484) and to the reference decompressor's output, raw bytes.
"""
import os
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
CLI = ROOT / "integration" / "_build" / "mgrc-gpu"


@pytest.fixture(scope="module")
def cli():
    if not CLI.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "integration"), "cli"], check=True)
    return str(CLI)


def run(cli, *args):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=600)


def test_usage_errors(cli):
    assert run(cli).returncode != 0
    r = run(cli, "compress", "--input", "x")
    assert r.returncode != 0 and "required" in r.stderr
    r = run(cli, "compress", "--bogus", "1")
    assert r.returncode != 0 and "unknown option" in r.stderr
    r = run(cli, "frobnicate")
    assert r.returncode != 0
    r = run(cli, "refactor", "--input", "a")
    assert r.returncode == 1 and r.stderr.startswith("error: InvalidState")


def test_size_mismatch(cli, tmp_path):
    f = tmp_path / "u.raw"
    np.zeros(100, dtype=np.float64).tofile(f)
    r = run(cli, "compress", "--input", f, "--output", tmp_path / "o", "--shape", "10x11", "--tol", "1e-3")
    assert r.returncode == 1
    assert r.stderr.strip() == (f"error: InvalidShape: size mismatch: {f} has 800 bytes, shape 10x11 needs 880")
    r = run(cli, "compress", "--input", f, "--output", tmp_path / "o", "--shape", "10xx10", "--tol", "1e-3")
    assert r.returncode == 1 and "InvalidShape: bad --shape" in r.stderr


def test_inspect_multiblock(cli, oracle, tmp_path):
    u = oracle.multisine_noisy((40, 33, 17), 42, 0.05).astype(np.float32)
    stream = oracle.compress_chunked(u, 1e-4, 0, 0.0, 1, 2, chunk_mem=17 * 33 * 17 * 4)
    p = tmp_path / "s.mgrc"
    p.write_bytes(stream)
    count = struct.unpack_from("<I", stream, 0)[0]
    offs = list(struct.unpack_from(f"<{count}Q", stream, 4)) + [len(stream)]
    want = f"format: mgrc-multiblock\nblocks: {count}\n"
    for i in range(count):
        want += f"--- block {i} ---\n" + oracle.describe(stream[offs[i]:offs[i + 1]])
    r = run(cli, "inspect", p)
    assert r.returncode == 0, r.stderr
    assert r.stdout == want
    # corrupt offsets / truncation (mgrc.cpp:277-293)
    bad = bytearray(stream)
    bad[4:12] = struct.pack("<Q", 3)
    p.write_bytes(bytes(bad))
    r = run(cli, "inspect", p)
    assert r.returncode == 1 and r.stderr.strip() == "error: CorruptStream: bad block offsets"
    p.write_bytes(stream[:6])
    r = run(cli, "inspect", p)
    assert r.returncode == 1 and "CorruptStream: truncated stream" in r.stderr


CASES = [
    # shape, dtype, tol, s, mode, chunk-mem argument (as typed), budget in bytes
    ((40, 33, 17), np.float32, 1e-4, "inf", "rel", "38148", 17 * 33 * 17 * 4),
    ((70, 65), np.float64, 1e-3, "inf", "abs", "20KiB", 20 * 1024),
    ((60, 20, 20), np.float64, 1e-3, "0", "rel", str(17 * 400 * 8), 17 * 400 * 8),
    ((33, 17), np.float64, 1e-3, "inf", "rel", None, 0),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[0])))
def test_cli_round_trip(cli, oracle, tmp_path, case):
    shape, dt, tol, s, mode, cm_text, cm = case
    u = oracle.multisine_noisy(shape, 42, 0.05).astype(dt)
    raw = tmp_path / "u.raw"
    u.tofile(raw)
    out = tmp_path / "u.mgrc"
    args = ["compress", "--input", raw, "--output", out, "--shape", "x".join(map(str, shape)),
            "--dtype", "f32" if dt == np.float32 else "f64", "--tol", repr(tol), "--s", s, "--mode", mode]
    if cm_text:
        args += ["--chunk-mem", cm_text]
    r = run(cli, *args)
    assert r.returncode == 0, r.stderr
    norm, sm = (0, 0.0) if s == "inf" else (1, float(s))
    want = oracle.compress_chunked(u, tol, norm, sm, 1 if mode == "rel" else 0, 2, chunk_mem=cm)
    got = out.read_bytes()
    assert got == want
    count = struct.unpack_from("<I", want, 0)[0]
    assert r.stderr.startswith(f"compressed {raw} ({u.nbytes} bytes) -> {out} ({len(want)} bytes), {count} block(s)")
    back = tmp_path / "back.raw"
    r = run(cli, "decompress", "--input", out, "--output", back)
    assert r.returncode == 0, r.stderr
    offs = list(struct.unpack_from(f"<{count}Q", want, 4)) + [len(want)]
    ref = np.concatenate([oracle.decompress(want[offs[i]:offs[i + 1]]) for i in range(count)], axis=0)
    assert back.read_bytes() == ref.astype(dt).tobytes()
    # the same stream and output from several GPU ranks of one process (--gpus; ranks share the device here)
    out3 = tmp_path / "u3.mgrc"
    r = run(cli, *[str(x) if x != out else out3 for x in args], "--gpus", "3")
    assert r.returncode == 0, r.stderr
    assert out3.read_bytes() == want
    back3 = tmp_path / "back3.raw"
    r = run(cli, "decompress", "--input", out3, "--output", back3, "--gpus", "2")
    assert r.returncode == 0, r.stderr
    assert back3.read_bytes() == back.read_bytes()


@pytest.mark.gpu
def test_cli_coords_and_codec(cli, oracle, tmp_path):
    shape = (40, 20)
    u = oracle.multisine_noisy(shape, 42, 0.05)
    coords = [np.cumsum(np.linspace(0.5, 1.5, n)) for n in shape]
    raw, cf, out = tmp_path / "u.raw", tmp_path / "c.f64", tmp_path / "u.mgrc"
    u.tofile(raw)
    np.concatenate(coords).astype(np.float64).tofile(cf)
    r = run(cli, "compress", "--input", raw, "--output", out, "--shape", "40x20", "--tol", "1e-3", "--codec", "1",
            "--coords", cf, "--chunk-mem", str(17 * 20 * 8))
    assert r.returncode == 0, r.stderr
    want = oracle.compress_chunked(u, 1e-3, 0, 0.0, 0, 1, chunk_mem=17 * 20 * 8, coords=coords)
    assert out.read_bytes() == want
    bad = tmp_path / "bad.f64"
    np.zeros(10).tofile(bad)
    r = run(cli, "compress", "--input", raw, "--output", out, "--shape", "40x20", "--tol", "1e-3", "--coords", bad)
    assert r.returncode == 1 and "coordinate file must hold 60 f64 values" in r.stderr

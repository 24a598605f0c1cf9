"""CPU tests of the C-ABI boundary (include/mgrc_gpu.h) — no compute calls.

* libmgrc_gpu.so loads and exports every entry point the header declares;
* the host-only entry points (inspect / describe / plan_chunks) agree with the
  reference on the golden fixtures;
* compute entry points fail loudly (MGRC_E_CUDA) when no CUDA device exists:
  the product path has no CPU fallback.
"""
import json
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import HAVE_CUDA

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "mgrc_gpu.h"
GOLD = ROOT / "tests" / "golden"
MAN = json.loads((GOLD / "manifest.json").read_text())


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"MGRC_GPU_API\s+[\w\s\*]+?\b(mgrc_gpu_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ["mgrc_gpu_compress", "mgrc_gpu_decompress", "mgrc_gpu_inspect", "mgrc_gpu_describe",
                 "mgrc_gpu_plan_chunks", "mgrc_gpu_compress_chunked", "mgrc_gpu_decompress_chunked",
                 "mgrc_gpu_last_error", "mgrc_gpu_free"]:
        assert must in syms


def test_library_exports_every_declared_symbol(mg):
    from paper_2401_05994_b200 import _lib

    L = _lib.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_library_is_sm100a():
    import subprocess

    so = ROOT / "paper_2401_05994_b200" / "libmgrc_gpu.so"
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    assert "sm_100a" in r.stdout


@pytest.mark.parametrize("case", MAN["containers"], ids=lambda c: c["name"])
def test_inspect_describe_match_reference(mg, case):
    blob = (GOLD / f"{case['name']}.mgrc").read_bytes()
    info = mg.inspect(blob)
    assert list(info.shape) == case["shape"]
    assert info.codec_id == case["codec"]
    assert info.header_size + info.payload_len == len(blob)
    assert mg.describe(info) == case["describe"]


def test_plan_chunks_match_reference(mg):
    for p in MAN["components"]["plans"]:
        got = mg.plan_chunks(tuple(p["shape"]), mg.DType(p["dtype"]), p["budget"])
        assert got.tolist() == p["blocks"]


def test_inspect_errors(mg):
    blob = (GOLD / "noisy_17_f64_inf_rel1e-3.mgrc").read_bytes()
    with pytest.raises(mg.MgrcError) as e:
        mg.inspect(b"XGRC" + blob[4:])
    assert e.value.name == "BadMagic"
    with pytest.raises(mg.MgrcError) as e:
        mg.inspect(blob[:10])
    assert e.value.name == "CorruptStream"
    b = bytearray(blob)
    b[4] = 9
    with pytest.raises(mg.MgrcError) as e:
        mg.inspect(bytes(b))
    assert e.value.name == "UnsupportedVersion"


@pytest.mark.skipif(HAVE_CUDA, reason="checks the no-device behaviour")
def test_compute_entry_points_fail_loudly_without_gpu(mg):
    u = np.linspace(0, 1, 17)
    with pytest.raises(mg.MgrcError) as e:
        mg.compress(u, mg.make_grid(u.shape), mg.ErrorSpec(1e-3))
    assert e.value.code == 100
    blob = (GOLD / "noisy_17_f64_inf_rel1e-3.mgrc").read_bytes()
    with pytest.raises(mg.MgrcError) as e:
        mg.decompress(blob)
    assert e.value.code == 100

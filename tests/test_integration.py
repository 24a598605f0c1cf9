"""The reference-side binding (integration/container_gpu.cpp): the reference's
own public API (mgrc::compress / decompress / inspect / describe with the
container.hpp signatures) running on the B200 path.

CPU: the binding compiles against the reference headers.  GPU: a client built
from the reference's own sources with container.cpp replaced by the binding
(integration/_build/mgrc_gpu_driver) produces the reference's container bytes
and decompressed values.
"""
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_INC = Path("/root/reference/proj/include")
DRIVER = ROOT / "integration" / "_build" / "mgrc_gpu_driver"


@pytest.mark.skipif(not REF_INC.exists(), reason="reference headers not present (GPU box)")
def test_binding_compiles_against_reference_headers(tmp_path):
    r = subprocess.run(["g++", "-std=c++20", "-Wall", "-Wextra", "-Werror", "-fsyntax-only", f"-I{REF_INC}",
                        f"-I{ROOT / 'include'}", str(ROOT / "integration" / "container_gpu.cpp")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
@pytest.mark.skipif(not DRIVER.exists(), reason="integration driver not built")
@pytest.mark.parametrize("shape,dt,tol,norm,s,mode", [
    ((65, 65, 65), "f64", 1e-3, "inf", 0.0, "rel"),
    ((33, 40, 21), "f32", 1e-4, "inf", 0.0, "rel"),
    ((129, 130), "f64", 1e-3, "s", 1.0, "rel"),
])
def test_reference_api_on_gpu(oracle, tmp_path, shape, dt, tol, norm, s, mode):
    u = oracle.multisine_noisy(shape, 42, 0.05).astype(np.float32 if dt == "f32" else np.float64)
    raw = tmp_path / "u.raw"
    u.tofile(raw)
    out = tmp_path / "u.mgrc"
    r = subprocess.run([str(DRIVER), "compress", str(raw), dt, str(tol), norm, str(s), mode, str(out),
                        *map(str, shape)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    want = oracle.compress(u, tol, 0 if norm == "inf" else 1, s, 0 if mode == "abs" else 1, 2)
    assert out.read_bytes() == want
    assert r.stdout == oracle.describe(want)
    back = tmp_path / "back.raw"
    r = subprocess.run([str(DRIVER), "decompress", str(out), str(back)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert back.read_bytes() == oracle.decompress(want).tobytes()

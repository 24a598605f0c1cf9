#!/usr/bin/env python3
"""Generates the golden fixtures under tests/golden/ from the REFERENCE itself.

TEST INFRASTRUCTURE.  Runs the unmodified reference library
(/root/reference/proj/src compiled in place by oracle/Makefile into
oracle/_ref/libmgrc_ref.so, with the reference's own test generators from
proj/tests/support/test_support.hpp) and records, per case:

  * sha256 of the input field (so the restated generators are pinned too),
  * the full container bytes (``<case>.mgrc``),
  * sha256 of the reference decompressor's output,
  * component outputs (forward coefficients, quantised codes, Huffman bytes,
    CRC values, chunk plans) as sha256 digests or small literal values.

Usage (in the build container, where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle import binding  # noqa: E402

# (name, shape, field, dtype, tol, norm, s, mode, codec, coords_seed)
CONTAINER_CASES = [
    ("cfg1_65c_f64_inf_rel1e-3", (65, 65, 65), "multisine", "f64", 1e-3, 0, 0.0, 1, 2, None),
    ("cfg1_65c_f64_s0_rel1e-3", (65, 65, 65), "multisine", "f64", 1e-3, 1, 0.0, 1, 2, None),
    ("noisy_33x17x9_f32_inf_rel1e-4", (33, 17, 9), "noisy", "f32", 1e-4, 0, 0.0, 1, 2, None),
    ("noisy_129x130_f64_s1_rel1e-3", (129, 130), "noisy", "f64", 1e-3, 1, 1.0, 1, 2, None),
    ("noisy_129x130_f64_s0_rel1e-3", (129, 130), "noisy", "f64", 1e-3, 1, 0.0, 1, 2, None),
    ("noisy_257x256_f32_inf_rel1e-5", (257, 256), "noisy", "f32", 1e-5, 0, 0.0, 1, 2, None),
    ("noisy_12x7x10_f32_s0_abs1e-3", (12, 7, 10), "noisy", "f32", 1e-3, 1, 0.0, 0, 2, None),
    ("noisy_6x5x4x3_f64_inf_abs1e-2", (6, 5, 4, 3), "noisy", "f64", 1e-2, 0, 0.0, 0, 2, None),
    ("noisy_17_f64_inf_rel1e-3", (17,), "noisy", "f64", 1e-3, 0, 0.0, 1, 2, None),
    ("noisy_2x2_f64_inf_abs1e-3", (2, 2), "noisy", "f64", 1e-3, 0, 0.0, 0, 2, None),
    ("random_100x3x40_f64_inf_abs1e-6", (100, 3, 40), "random", "f64", 1e-6, 0, 0.0, 0, 2, None),
    ("random_65x65_f64_inf_abs1e-14", (65, 65), "random", "f64", 1e-14, 0, 0.0, 0, 2, None),
    ("noisy_33x20_f64_codec1", (33, 20), "noisy", "f64", 1e-3, 0, 0.0, 1, 1, None),
    ("noisy_33x20_f32_codec0", (33, 20), "noisy", "f32", 1e-3, 0, 0.0, 1, 0, None),
    ("coords_17x12x9_f64_inf_abs1e-3", (17, 12, 9), "noisy", "f64", 1e-3, 0, 0.0, 0, 2, 3),
    ("const_9x33_f64", (9, 33), "const3.25", "f64", 1e-3, 0, 0.0, 1, 2, None),
    ("const_9x33_f64_negzero", (9, 33), "const-0.0", "f64", 1e-3, 0, 0.0, 1, 2, None),
]

# chunked (multiblock) streams: (name, shape, field, dtype, tol, norm, s, mode, chunk_mem)
CHUNKED_CASES = [
    ("chunked_40x33x17_f32_inf_rel1e-4", (40, 33, 17), "multisine", "f32", 1e-4, 0, 0.0, 1, 17 * 33 * 17 * 4),
    ("chunked_70x65_f64_inf_abs1e-3", (70, 65), "noisy", "f64", 1e-3, 0, 0.0, 0, 20 * 65 * 8),
]

PLAN_CASES = [
    ((2049, 2049, 2049), 0, 257 * 2049 * 2049 * 4),
    ((2049, 2049, 2049), 0, 129 * 2049 * 2049 * 4),
    ((2049, 2049, 2049), 0, 2049 ** 3 * 4 // 8),
    ((513, 513, 513), 0, 513 ** 3 * 4 // 3),
    ((100, 70), 1, 17 * 70 * 8),
    ((40, 33, 17), 0, 17 * 33 * 17 * 4),
]


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


def fib_stream(nsym=22):
    """A byte stream whose symbol counts are Fibonacci numbers: the natural
    Huffman tree has depth nsym-1 > 15, so build_lengths' Kraft repair
    (codec.cpp:157-190) is exercised."""
    f = [1, 1]
    while len(f) < nsym:
        f.append(f[-1] + f[-2])
    syms = np.concatenate([np.full(c, (37 * k + 11) & 0xFF, np.uint8) for k, c in enumerate(f)])
    rng = np.random.default_rng(5)
    rng.shuffle(syms)
    return syms.tobytes()


def main():
    ref = binding.get("reference")
    ref.set_threads(1)
    man = {"generator": "oracle/_ref/libmgrc_ref.so (reference sources compiled unmodified)",
           "containers": [], "chunked": [], "components": {}}
    for name, shape, kind, dt, tol, norm, s, mode, codec, cseed in CONTAINER_CASES:
        u = make_field(ref, kind, shape, dt)
        coords = make_coords(shape, cseed) if cseed is not None else None
        blob = ref.compress(u, tol, norm, s, mode, codec, coords=coords)
        back = ref.decompress(blob)
        (HERE / f"{name}.mgrc").write_bytes(blob)
        man["containers"].append({
            "name": name, "shape": list(shape), "field": kind, "dtype": dt, "tol": tol, "norm": norm, "s": s,
            "mode": mode, "codec": codec, "coords_seed": cseed, "input_sha256": sha(u), "container_len": len(blob),
            "container_sha256": sha(blob), "output_sha256": sha(back), "describe": ref.describe(blob),
        })
    for name, shape, kind, dt, tol, norm, s, mode, cm in CHUNKED_CASES:
        u = make_field(ref, kind, shape, dt)
        blob = ref.compress_chunked(u, tol, norm, s, mode, 2, chunk_mem=cm)
        (HERE / f"{name}.mgrcm").write_bytes(blob)
        man["chunked"].append({"name": name, "shape": list(shape), "field": kind, "dtype": dt, "tol": tol,
                               "norm": norm, "s": s, "mode": mode, "chunk_mem": cm, "input_sha256": sha(u),
                               "stream_sha256": sha(blob), "stream_len": len(blob)})
    comp = man["components"]
    # transform / quantise digests on the reference's own generators
    for shape in [(17,), (6,), (9, 5), (33, 17, 9), (12, 7, 10), (6, 5, 4, 3), (65, 65, 65), (257, 256)]:
        u = ref.multisine_noisy(shape, 42, 0.05)
        c = ref.forward(u)
        key = "x".join(map(str, shape))
        h = ref.hierarchy(shape)
        L = h["nlevels"]
        tau = ref.absolute_tolerance(u, 1e-3, 0, 0.0, 1)
        w = ref.bin_widths(tau, 0, 0.0, len(shape), L)
        q, r, outl = ref.quantize(c, w)
        comp[f"forward:{key}"] = sha(c)
        comp[f"inverse_of_forward:{key}"] = sha(ref.inverse(c))
        comp[f"quantize_q:{key}"] = sha(q)
        comp[f"quantize_r:{key}"] = sha(r)
        comp[f"nlevels:{key}"] = L
        comp[f"node_counts:{key}"] = [int(x) for x in h["node_counts"]]
    fs = fib_stream()
    packed = ref.huffman_pack(fs)
    (HERE / "huffman_fib22.bin").write_bytes(fs)
    comp["huffman_fib22_packed_sha256"] = sha(packed)
    comp["huffman_fib22_packed_len"] = len(packed)
    comp["huffman_fib22_table_header_hex"] = packed[:131].hex()
    for data in [b"", b"123456789", b"The quick brown fox jumps over the lazy dog", bytes(range(256)) * 7]:
        comp[f"crc32:{sha(data)[:16]}"] = ref.crc32(data)
    v = np.array([0, 0, 0, 0, -1, 1, 63, -64, 64, 8191, -8192, 2 ** 40, -(2 ** 62), 2 ** 63 - 1, -(2 ** 63)],
                 dtype=np.int64)
    for codec in (0, 1, 2):
        comp[f"lossless_encode:codec{codec}"] = ref.lossless_encode(v, codec).hex()
    plans = []
    for shape, dt, budget in PLAN_CASES:
        p = ref.plan_chunks(shape, dt, budget)
        plans.append({"shape": list(shape), "dtype": dt, "budget": budget, "blocks": p.tolist()})
    comp["plans"] = plans
    (HERE / "manifest.json").write_text(json.dumps(man, indent=1) + "\n")
    total = sum(p.stat().st_size for p in HERE.iterdir())
    print(f"wrote {len(man['containers'])} containers, {len(man['chunked'])} chunked streams; {total / 1e6:.2f} MB")


if __name__ == "__main__":
    main()

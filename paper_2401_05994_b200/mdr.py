"""MDR refactor / recompose (row f2): progressive retrieval by (level, bitplane)
segments, mirroring ``/root/reference/proj/include/mgrc/refactor.hpp:81-117``.

    store = refactor(u, grid, planes=32)              # refactor.cpp:144-218 (GPU)
    write_store(store, "dir")                          # manifest.json + l{L}_b{P}.bin files
    m = read_manifest("dir")
    req = request(m, tol_abs=1e-3, norm=Norm.inf)      # greedy planner (refactor.cpp:226-272)
    st = make_initial_state(m)
    u1 = reconstruct(m, directory_source("dir", m), req, st)   # refactor.cpp:274-357 (GPU)
    req2 = request(m, 1e-5, Norm.inf, state=st)        # refine: only the missing segments
    u2 = reconstruct(m, directory_source("dir", m), req2, st)

The segments are byte-identical to the reference's (same fixed point, same
bit planes, same canonical Huffman tables, same CRC-32); the plan is the
reference's; the reconstruction is bit-identical to the reference's.  The
manifest JSON carries the reference's fields (``manifest_to_json``), so either
side reads the other's stores.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import struct
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import Norm, TensorGrid, _check, _f64_ptr, _grid_args, _is_torch, _lib, _take, make_grid

INT32_MIN = -(1 << 31)


class ManifestC(C.Structure):
    _fields_ = [("ndims", C.c_int), ("shape", C.c_uint64 * 4), ("nlevels", C.c_int), ("planes", C.c_uint32),
                ("level_exponents", C.c_int32 * 65), ("level_counts", C.c_uint64 * 65),
                ("value_min", C.c_double), ("value_max", C.c_double), ("value_rms", C.c_double)]


class SegmentC(C.Structure):
    _fields_ = [("bytes", C.c_uint64), ("raw_bits", C.c_uint64), ("crc32", C.c_uint32)]


_SIGS = {
    "mgrc_gpu_mdr_refactor": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_uint32,
                                        C.POINTER(C.c_void_p)]),
    "mgrc_gpu_mdr_store_manifest": (C.c_int, [C.c_void_p, C.POINTER(ManifestC), C.c_void_p]),
    "mgrc_gpu_mdr_store_segment": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p),
                                             C.POINTER(C.c_uint64)]),
    "mgrc_gpu_mdr_store_free": (None, [C.c_void_p]),
    "mgrc_gpu_mdr_request": (C.c_int, [C.POINTER(ManifestC), C.c_void_p, C.c_double, C.c_int, C.c_double,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    "mgrc_gpu_mdr_session_new": (C.c_int, [C.POINTER(ManifestC), C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "mgrc_gpu_mdr_reconstruct": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                           C.c_int, C.c_double, C.c_void_p, C.POINTER(C.c_double), C.c_void_p]),
    "mgrc_gpu_mdr_session_free": (None, [C.c_void_p]),
}


def _L():
    L = _lib.lib()
    if not getattr(L, "_mdr_ready", False):
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        L._mdr_ready = True
    return L


@dataclass
class SegmentMeta:  # refactor.hpp:26-31
    byte_size: int
    raw_bits: int
    checksum: int
    file_name: str


@dataclass
class StoreManifest:  # refactor.hpp:33-45
    shape: Tuple[int, ...]
    coords: Optional[List[np.ndarray]]
    nlevels: int
    planes: int
    level_exponents: List[Optional[int]]  # None: empty level
    level_counts: List[int]
    value_min: float
    value_max: float
    value_rms: float
    segments: List[List[SegmentMeta]]
    dtype: str = "f64"

    def grid(self) -> TensorGrid:
        return make_grid(self.shape, self.coords)

    def _c(self):
        m = ManifestC()
        m.ndims = len(self.shape)
        for a, n in enumerate(self.shape):
            m.shape[a] = n
        m.nlevels = self.nlevels
        m.planes = self.planes
        for l in range(self.nlevels + 1):
            e = self.level_exponents[l]
            m.level_exponents[l] = INT32_MIN if e is None else e
            m.level_counts[l] = self.level_counts[l]
        m.value_min, m.value_max, m.value_rms = self.value_min, self.value_max, self.value_rms
        segs = (SegmentC * ((self.nlevels + 1) * self.planes))()
        for l in range(self.nlevels + 1):
            for p in range(self.planes):
                s = self.segments[l][p]
                segs[l * self.planes + p] = SegmentC(s.byte_size, s.raw_bits, s.checksum)
        return m, segs


@dataclass
class RefactoredStore:  # refactor.hpp:50-53
    manifest: StoreManifest
    segments: List[List[bytes]]


@dataclass
class SegmentRequest:  # refactor.hpp:64-69
    segments: List[Tuple[int, int]]
    predicted: float
    satisfiable: bool
    total_bytes: int


@dataclass
class RetrievalState:  # refactor.hpp:56-62: the accumulators live on the GPU (one session per state)
    planes_fetched: List[int]
    accrued: float = float("inf")
    _session: Optional[int] = field(default=None, repr=False)
    _keep: object = field(default=None, repr=False)

    def __del__(self):
        if self._session:
            _L().mgrc_gpu_mdr_session_free(self._session)
            self._session = None


def refactor(u, grid: Optional[TensorGrid] = None, planes: int = 32) -> RefactoredStore:
    """refactor (refactor.cpp:144-218) on the GPU: f64 input (numpy or torch, host or CUDA)."""
    L = _L()
    ptr, shape, keep = _f64_ptr(u, "u")
    grid = grid or make_grid(shape)
    gshape, coords, ck = _grid_args(grid)
    h = C.c_void_p()
    _check(L.mgrc_gpu_mdr_refactor(ptr, len(gshape), gshape.ctypes.data, coords, planes, C.byref(h)))
    try:
        mc = ManifestC()
        _check(L.mgrc_gpu_mdr_store_manifest(h, C.byref(mc), None))
        nl, B = mc.nlevels, mc.planes
        segs_c = (SegmentC * ((nl + 1) * B))()
        _check(L.mgrc_gpu_mdr_store_manifest(h, C.byref(mc), segs_c))
        segs, payload = [], []
        for l in range(nl + 1):
            row, prow = [], []
            for p in range(B):
                s = segs_c[l * B + p]
                row.append(SegmentMeta(int(s.bytes), int(s.raw_bits), int(s.crc32), f"l{l}_b{p}.bin"))
                d, n = C.c_void_p(), C.c_uint64()
                _check(L.mgrc_gpu_mdr_store_segment(h, l, p, C.byref(d), C.byref(n)))
                prow.append(bytes(_take(d, n.value)) if n.value else b"")
            segs.append(row)
            payload.append(prow)
        m = StoreManifest(
            shape=tuple(int(mc.shape[a]) for a in range(mc.ndims)),
            coords=None if grid.coords is None else [np.asarray(c, np.float64) for c in grid.coords],
            nlevels=nl, planes=B,
            level_exponents=[None if mc.level_exponents[l] == INT32_MIN else int(mc.level_exponents[l])
                             for l in range(nl + 1)],
            level_counts=[int(mc.level_counts[l]) for l in range(nl + 1)],
            value_min=mc.value_min, value_max=mc.value_max, value_rms=mc.value_rms, segments=segs)
        return RefactoredStore(m, payload)
    finally:
        L.mgrc_gpu_mdr_store_free(h)


def make_initial_state(manifest: StoreManifest) -> RetrievalState:
    """make_initial_state (refactor.cpp:210-221)."""
    return RetrievalState([0] * (manifest.nlevels + 1))


def request(manifest: StoreManifest, tol_abs: float, norm: Norm = Norm.inf, smoothness: float = 0.0,
            state: Optional[RetrievalState] = None) -> SegmentRequest:
    """request (refactor.cpp:226-272): the greedy plan from `state`."""
    L = _L()
    m, segs = manifest._c()
    fetched = np.asarray(state.planes_fetched if state else [0] * (manifest.nlevels + 1), dtype=np.uint32)
    cap = (manifest.nlevels + 1) * manifest.planes
    lv = np.zeros(cap, dtype=np.uint32)
    pl = np.zeros(cap, dtype=np.uint32)
    n, by, pred, sat = C.c_uint64(), C.c_uint64(), C.c_double(), C.c_int()
    _check(L.mgrc_gpu_mdr_request(C.byref(m), segs, tol_abs, int(norm), smoothness, fetched.ctypes.data,
                                  lv.ctypes.data, pl.ctypes.data, cap, C.byref(n), C.byref(by), C.byref(pred),
                                  C.byref(sat)))
    return SegmentRequest([(int(lv[i]), int(pl[i])) for i in range(n.value)], pred.value, bool(sat.value),
                          int(by.value))


def reconstruct(manifest: StoreManifest, source: Callable[[int, int], bytes], req: SegmentRequest,
                state: RetrievalState, norm: Norm = Norm.inf, smoothness: float = 0.0, out=None):
    """reconstruct (refactor.cpp:274-357) on the GPU: applies the request to `state` and returns the refined
    field (numpy, or into `out`: a host or CUDA float64 array of the grid's shape)."""
    L = _L()
    if state._session is None:
        m, segs = manifest._c()
        _, coords, ck = _grid_args(manifest.grid())
        h = C.c_void_p()
        _check(L.mgrc_gpu_mdr_session_new(C.byref(m), segs, coords, C.byref(h)))
        state._session = h.value
    payloads = [source(l, p) if manifest.level_exponents[l] is not None else b"" for l, p in req.segments]
    n = len(req.segments)
    bufs = [np.frombuffer(b, dtype=np.uint8) if b else np.zeros(1, np.uint8) for b in payloads]
    ptrs = (C.c_void_p * max(n, 1))(*[b.ctypes.data for b in bufs])
    lens = np.asarray([len(b) for b in payloads] or [0], dtype=np.uint64)
    lv = np.asarray([a for a, _ in req.segments] or [0], dtype=np.uint32)
    pl = np.asarray([b for _, b in req.segments] or [0], dtype=np.uint32)
    if out is None:
        out = np.empty(manifest.shape, dtype=np.float64)
    optr = out.data_ptr() if _is_torch(out) else out.ctypes.data
    acc = C.c_double()
    fetched = np.zeros(manifest.nlevels + 1, dtype=np.uint32)
    _check(L.mgrc_gpu_mdr_reconstruct(state._session, lv.ctypes.data, pl.ctypes.data, n, ptrs, lens.ctypes.data,
                                      int(norm), smoothness, optr, C.byref(acc), fetched.ctypes.data))
    state.planes_fetched = [int(x) for x in fetched]
    state.accrued = acc.value
    return out


# ---- persistence (refactor.cpp:359-549): manifest.json + one file per segment ----


def manifest_to_json(m: StoreManifest) -> str:
    """The reference's manifest document (refactor.cpp:368-401): the same fields in the same order."""
    j = {
        "format": "mgrc-store", "version": 1, "dtype": m.dtype, "shape": list(m.shape),
        "coords": None if m.coords is None else [[float(x) for x in c] for c in m.coords],
        "nlevels": m.nlevels, "planes": m.planes,
        "stats": {"min": m.value_min, "max": m.value_max, "rms": m.value_rms},
        "level_exponents": m.level_exponents, "level_counts": m.level_counts,
        "segments": [{"level": l, "plane": p, "bytes": s.byte_size, "bits": s.raw_bits, "crc32": s.checksum,
                      "file": s.file_name} for l, row in enumerate(m.segments) for p, s in enumerate(row)],
    }
    return json.dumps(j, indent=2) + "\n"


def manifest_from_json(text: str) -> StoreManifest:
    j = json.loads(text)
    if j.get("format") != "mgrc-store":
        from . import MgrcError

        raise MgrcError(10, "BadMagic: not an mgrc store manifest")
    nl, B = int(j["nlevels"]), int(j["planes"])
    segs = [[None] * B for _ in range(nl + 1)]
    for s in j["segments"]:
        segs[int(s["level"])][int(s["plane"])] = SegmentMeta(int(s["bytes"]), int(s["bits"]), int(s["crc32"]),
                                                             s["file"])
    return StoreManifest(
        shape=tuple(int(x) for x in j["shape"]),
        coords=None if j["coords"] is None else [np.asarray(c, np.float64) for c in j["coords"]],
        nlevels=nl, planes=B, level_exponents=[None if e is None else int(e) for e in j["level_exponents"]],
        level_counts=[int(x) for x in j["level_counts"]], value_min=float(j["stats"]["min"]),
        value_max=float(j["stats"]["max"]), value_rms=float(j["stats"]["rms"]), segments=segs, dtype=j["dtype"])


def write_store(store: RefactoredStore, directory) -> None:
    """write_store (refactor.hpp:99-102): manifest.json + l{level}_b{plane}.bin = u32 crc32 | u64 raw bit count |
    encoded payload."""
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    m = store.manifest
    for l, row in enumerate(m.segments):
        for p, s in enumerate(row):
            (d / s.file_name).write_bytes(struct.pack("<IQ", s.checksum, s.raw_bits) + store.segments[l][p])
    (d / "manifest.json").write_text(manifest_to_json(m))


def read_manifest(directory) -> StoreManifest:
    return manifest_from_json((Path(directory) / "manifest.json").read_text())


def directory_source(directory, manifest: StoreManifest) -> Callable[[int, int], bytes]:
    d = Path(directory)

    def src(level: int, plane: int) -> bytes:
        raw = (d / manifest.segments[level][plane].file_name).read_bytes()
        return raw[12:]

    return src

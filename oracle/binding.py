"""TEST INFRASTRUCTURE ONLY — ctypes binding to the CPU oracles.

Two interchangeable implementations of the same ``oc_*`` C API:

* ``restatement`` — ``oracle/liboracle.so``, the plain-C restatement of the
  reference path (``oracle/mgrc_oracle.c``), the parity checker;
* ``reference``   — ``oracle/_ref/libmgrc_ref.so``, the unmodified reference
  library compiled in place from ``/root/reference/proj/src`` (``oracle/Makefile``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this module.  The product path
(``paper_2401_05994_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIBS = {
    "restatement": HERE / "liboracle.so",
    "reference": HERE / "_ref" / "libmgrc_ref.so",
}

ERRC_NAMES = [
    "InvalidShape", "TooManyDims", "LevelOutOfRange", "ShapeMismatch", "NonFiniteInput",
    "DegenerateData", "Overflow", "UnknownCodec", "CorruptStream", "BadMagic",
    "UnsupportedVersion", "ChecksumMismatch", "ToleranceUnreachable", "PlaneCountOutOfRange",
    "UnsatisfiableTolerance", "InvalidState", "PrefixViolation", "BudgetTooSmall", "IoError",
]


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        self.name = ERRC_NAMES[code - 1] if 1 <= code <= len(ERRC_NAMES) else f"E{code}"
        super().__init__(msg)


class OcInfo(C.Structure):
    _fields_ = [
        ("version", C.c_uint16), ("constant_field", C.c_uint8), ("coords_present", C.c_uint8),
        ("dtype", C.c_uint8), ("ndims", C.c_uint8), ("nlevels", C.c_uint8), ("codec_id", C.c_uint8),
        ("shape", C.c_uint64 * 4), ("mode", C.c_uint8), ("norm", C.c_uint8),
        ("smoothness", C.c_double), ("tol", C.c_double), ("bin_widths", C.c_double * 65),
        ("payload_len", C.c_uint64), ("checksum", C.c_uint32), ("header_size", C.c_uint64),
    ]


P = C.c_void_p
U64P = C.POINTER(C.c_uint64)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(P)


def _shape_arr(shape):
    return np.ascontiguousarray(np.asarray(shape, dtype=np.uint64))


def _coords_arr(coords):
    if coords is None:
        return None
    return np.ascontiguousarray(np.concatenate([np.asarray(c, dtype=np.float64) for c in coords]))


class Oracle:
    """Same interface for the restatement and the compiled reference."""

    def __init__(self, kind: str = "restatement"):
        path = LIBS[kind]
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.kind = kind
        self.lib = L = C.CDLL(str(path))
        L.oc_last_error.restype = C.c_char_p
        L.oc_crc32.restype = C.c_uint32
        L.oc_crc32.argtypes = [P, C.c_uint64]
        L.oc_round_half_even.restype = C.c_double
        L.oc_round_half_even.argtypes = [C.c_double]
        L.oc_sum_squares.restype = C.c_double
        L.oc_sum_squares.argtypes = [P, C.c_uint64]
        L.oc_set_threads.argtypes = [C.c_int]
        L.oc_impl.restype = C.c_char_p
        L.oc_compress.argtypes = [P, C.c_int, C.c_int, P, P, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int,
                                  C.POINTER(P), U64P]
        L.oc_compress_chunked.argtypes = [P, C.c_int, C.c_int, P, P, C.c_double, C.c_int, C.c_double, C.c_int,
                                          C.c_int, C.c_uint64, C.POINTER(P), U64P]
        L.oc_decompress.argtypes = [P, C.c_uint64, C.POINTER(P), C.POINTER(C.c_int), C.POINTER(C.c_int), P]
        L.oc_inspect.argtypes = [P, C.c_uint64, C.POINTER(OcInfo)]
        L.oc_describe.argtypes = [P, C.c_uint64, C.POINTER(C.c_char_p)]
        L.oc_free.argtypes = [P]
        L.oc_multisine.argtypes = [C.c_int, P, P]
        L.oc_random_field.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, P]
        L.oc_multisine_noisy.argtypes = [C.c_int, P, C.c_uint64, C.c_double, P]
        L.oc_mt19937_64.argtypes = [C.c_uint64, C.c_uint64, P]
        L.oc_hierarchy.argtypes = [C.c_int, P, P, C.POINTER(C.c_int), P, P, P, C.c_int]
        L.oc_level_set.argtypes = [C.c_int, P, C.c_int, C.c_int, P, U64P]
        L.oc_forward.argtypes = [C.c_int, P, P, P, P]
        L.oc_inverse.argtypes = [C.c_int, P, P, P, P]
        L.oc_quantize.argtypes = [C.c_int, P, P, P, P, P, P, U64P]
        L.oc_dequantize.argtypes = [C.c_int, P, P, P, P, P]
        L.oc_absolute_tolerance.argtypes = [P, C.c_uint64, C.c_double, C.c_int, C.c_double, C.c_int,
                                            C.POINTER(C.c_double)]
        L.oc_bin_widths.argtypes = [C.c_double, C.c_int, C.c_double, C.c_int, C.c_int, P]
        L.oc_achieved_error.argtypes = [C.c_int, P, P, P, C.c_int, C.c_double, C.POINTER(C.c_double)]
        L.oc_huffman_pack.argtypes = [P, C.c_uint64, C.POINTER(P), U64P]
        L.oc_huffman_unpack.argtypes = [P, C.c_uint64, C.c_uint64, P]
        L.oc_lossless_encode.argtypes = [P, C.c_uint64, C.c_int, C.POINTER(P), U64P]
        L.oc_lossless_decode.argtypes = [P, C.c_uint64, C.c_uint64, C.c_int, P]
        L.oc_plan_chunks.argtypes = [C.c_int, P, C.c_int, C.c_uint64, U64P, P, C.c_uint64]

    # -- helpers --------------------------------------------------------
    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.oc_last_error().decode())

    def _take_bytes(self, p, n):
        b = bytes((C.c_uint8 * n).from_address(p.value if hasattr(p, "value") else p)) if n else b""
        self.lib.oc_free(p)
        return b

    def set_threads(self, n: int) -> int:
        return self.lib.oc_set_threads(n)

    # -- container pipeline --------------------------------------------
    def compress(self, u, tol, norm=0, s=0.0, mode=0, codec=2, coords=None, shape=None) -> bytes:
        u = np.ascontiguousarray(u)
        dtype = 0 if u.dtype == np.float32 else 1
        if dtype == 1:
            u = np.ascontiguousarray(u, dtype=np.float64)
        shape = _shape_arr(u.shape if shape is None else shape)
        cs = _coords_arr(coords)
        out = P()
        n = C.c_uint64()
        self._check(self.lib.oc_compress(_ptr(u), dtype, len(shape), _ptr(shape), _ptr(cs), tol, norm, s, mode,
                                         codec, C.byref(out), C.byref(n)))
        return self._take_bytes(out, n.value)

    def compress_chunked(self, u, tol, norm=0, s=0.0, mode=0, codec=2, chunk_mem=0, coords=None) -> bytes:
        u = np.ascontiguousarray(u)
        dtype = 0 if u.dtype == np.float32 else 1
        shape = _shape_arr(u.shape)
        cs = _coords_arr(coords)
        out = P()
        n = C.c_uint64()
        self._check(self.lib.oc_compress_chunked(_ptr(u), dtype, len(shape), _ptr(shape), _ptr(cs), tol, norm, s,
                                                 mode, codec, chunk_mem, C.byref(out), C.byref(n)))
        return self._take_bytes(out, n.value)

    def decompress(self, blob: bytes) -> np.ndarray:
        buf = np.frombuffer(blob, dtype=np.uint8)
        out = P()
        dt = C.c_int()
        nd = C.c_int()
        shape = np.zeros(4, dtype=np.uint64)
        self._check(self.lib.oc_decompress(_ptr(buf), len(blob), C.byref(out), C.byref(dt), C.byref(nd),
                                           _ptr(shape)))
        sh = tuple(int(x) for x in shape[: nd.value])
        npdt = np.float32 if dt.value == 0 else np.float64
        cnt = int(np.prod(sh))
        nb = cnt * np.dtype(npdt).itemsize  # (ctypes.string_at truncates sizes beyond 2 GiB)
        arr = np.frombuffer((C.c_uint8 * nb).from_address(out.value), dtype=npdt).reshape(sh).copy()
        self.lib.oc_free(out)
        return arr

    def inspect(self, blob: bytes) -> OcInfo:
        buf = np.frombuffer(blob, dtype=np.uint8)
        info = OcInfo()
        self._check(self.lib.oc_inspect(_ptr(buf), len(blob), C.byref(info)))
        return info

    def describe(self, blob: bytes) -> str:
        buf = np.frombuffer(blob, dtype=np.uint8)
        t = C.c_char_p()
        self._check(self.lib.oc_describe(_ptr(buf), len(blob), C.byref(t)))
        s = t.value.decode()
        self.lib.oc_free(C.cast(t, P))
        return s

    # -- components ------------------------------------------------------
    def hierarchy(self, shape, coords=None):
        shape = _shape_arr(shape)
        cs = _coords_arr(coords)
        L = C.c_int()
        al = np.zeros(int(shape.sum()), dtype=np.uint8)
        nc = np.zeros(65, dtype=np.uint64)
        ls = np.zeros(65 * len(shape), dtype=np.uint64)
        self._check(self.lib.oc_hierarchy(len(shape), _ptr(shape), _ptr(cs), C.byref(L), _ptr(al), _ptr(nc),
                                          _ptr(ls), 65))
        Lv = L.value
        splits = np.cumsum(shape)[:-1].astype(np.int64)
        return {
            "nlevels": Lv,
            "axis_level": [a.copy() for a in np.split(al, splits)],
            "node_counts": nc[: Lv + 1].copy(),
            "level_shapes": ls[: (Lv + 1) * len(shape)].reshape(Lv + 1, len(shape)).copy(),
        }

    def level_set(self, shape, level, axis):
        shape = _shape_arr(shape)
        n = C.c_uint64()
        self._check(self.lib.oc_level_set(len(shape), _ptr(shape), level, axis, None, C.byref(n)))
        out = np.zeros(n.value, dtype=np.uint64)
        self._check(self.lib.oc_level_set(len(shape), _ptr(shape), level, axis, _ptr(out), C.byref(n)))
        return out

    def forward(self, u, coords=None):
        u = np.ascontiguousarray(u, dtype=np.float64)
        shape = _shape_arr(u.shape)
        out = np.empty_like(u)
        self._check(self.lib.oc_forward(len(shape), _ptr(shape), _ptr(_coords_arr(coords)), _ptr(u), _ptr(out)))
        return out

    def inverse(self, c, coords=None):
        c = np.ascontiguousarray(c, dtype=np.float64)
        shape = _shape_arr(c.shape)
        out = np.empty_like(c)
        self._check(self.lib.oc_inverse(len(shape), _ptr(shape), _ptr(_coords_arr(coords)), _ptr(c), _ptr(out)))
        return out

    def quantize(self, c, widths, coords=None):
        c = np.ascontiguousarray(c, dtype=np.float64)
        shape = _shape_arr(c.shape)
        w = np.ascontiguousarray(widths, dtype=np.float64)
        q = np.empty(c.shape, dtype=np.int64)
        r = np.empty_like(c)
        outl = C.c_uint64()
        self._check(self.lib.oc_quantize(len(shape), _ptr(shape), _ptr(_coords_arr(coords)), _ptr(c), _ptr(w),
                                         _ptr(q), _ptr(r), C.byref(outl)))
        return q, r, outl.value

    def dequantize(self, q, widths, coords=None):
        q = np.ascontiguousarray(q, dtype=np.int64)
        shape = _shape_arr(q.shape)
        w = np.ascontiguousarray(widths, dtype=np.float64)
        c = np.empty(q.shape, dtype=np.float64)
        self._check(self.lib.oc_dequantize(len(shape), _ptr(shape), _ptr(_coords_arr(coords)), _ptr(q), _ptr(w),
                                           _ptr(c)))
        return c

    def round_half_even(self, x: float) -> float:
        return self.lib.oc_round_half_even(x)

    def absolute_tolerance(self, u, tol, norm=0, s=0.0, mode=0) -> float:
        u = np.ascontiguousarray(u, dtype=np.float64).ravel()
        out = C.c_double()
        self._check(self.lib.oc_absolute_tolerance(_ptr(u), u.size, tol, norm, s, mode, C.byref(out)))
        return out.value

    def bin_widths(self, tau, norm, s, ndims, nlevels):
        out = np.zeros(nlevels + 1, dtype=np.float64)
        self._check(self.lib.oc_bin_widths(tau, norm, s, ndims, nlevels, _ptr(out)))
        return out

    def achieved_error(self, res, norm=0, s=0.0, coords=None) -> float:
        res = np.ascontiguousarray(res, dtype=np.float64)
        shape = _shape_arr(res.shape)
        out = C.c_double()
        self._check(self.lib.oc_achieved_error(len(shape), _ptr(shape), _ptr(_coords_arr(coords)), _ptr(res), norm,
                                               s, C.byref(out)))
        return out.value

    def sum_squares(self, v) -> float:
        v = np.ascontiguousarray(v, dtype=np.float64).ravel()
        return self.lib.oc_sum_squares(_ptr(v), v.size)

    def crc32(self, data: bytes) -> int:
        buf = np.frombuffer(data, dtype=np.uint8)
        return self.lib.oc_crc32(_ptr(buf), len(data))

    def huffman_pack(self, data: bytes) -> bytes:
        buf = np.frombuffer(data, dtype=np.uint8)
        out = P()
        n = C.c_uint64()
        self._check(self.lib.oc_huffman_pack(_ptr(buf), len(data), C.byref(out), C.byref(n)))
        return self._take_bytes(out, n.value)

    def huffman_unpack(self, packed: bytes, count: int) -> bytes:
        buf = np.frombuffer(packed, dtype=np.uint8)
        out = np.zeros(max(count, 1), dtype=np.uint8)
        self._check(self.lib.oc_huffman_unpack(_ptr(buf), len(packed), count, _ptr(out)))
        return out[:count].tobytes()

    def lossless_encode(self, values, codec=2) -> bytes:
        v = np.ascontiguousarray(values, dtype=np.int64).ravel()
        out = P()
        n = C.c_uint64()
        self._check(self.lib.oc_lossless_encode(_ptr(v), v.size, codec, C.byref(out), C.byref(n)))
        return self._take_bytes(out, n.value)

    def lossless_decode(self, payload: bytes, count: int, codec=2):
        buf = np.frombuffer(payload, dtype=np.uint8)
        out = np.zeros(max(count, 1), dtype=np.int64)
        self._check(self.lib.oc_lossless_decode(_ptr(buf), len(payload), count, codec, _ptr(out)))
        return out[:count]

    def plan_chunks(self, shape, dtype, budget):
        shape = _shape_arr(shape)
        nb = C.c_uint64()
        self._check(self.lib.oc_plan_chunks(len(shape), _ptr(shape), dtype, budget, C.byref(nb), None, 0))
        out = np.zeros(int(nb.value) * len(shape) * 2, dtype=np.uint64)
        self._check(self.lib.oc_plan_chunks(len(shape), _ptr(shape), dtype, budget, C.byref(nb), _ptr(out),
                                            nb.value))
        return out.reshape(int(nb.value), len(shape), 2)

    # -- fields ------------------------------------------------------------
    def multisine(self, shape):
        shape_a = _shape_arr(shape)
        out = np.empty(tuple(int(s) for s in shape), dtype=np.float64)
        self.lib.oc_multisine(len(shape_a), _ptr(shape_a), _ptr(out))
        return out

    def multisine_noisy(self, shape, seed=42, noise=0.05):
        shape_a = _shape_arr(shape)
        out = np.empty(tuple(int(s) for s in shape), dtype=np.float64)
        self.lib.oc_multisine_noisy(len(shape_a), _ptr(shape_a), seed, noise, _ptr(out))
        return out

    def random_field(self, shape, seed, lo=-1.0, hi=1.0):
        n = int(np.prod(shape))
        out = np.empty(n, dtype=np.float64)
        self.lib.oc_random_field(n, seed, lo, hi, _ptr(out))
        return out.reshape(shape)

    def mt19937_64(self, seed, n):
        out = np.empty(n, dtype=np.uint64)
        self.lib.oc_mt19937_64(seed, n, _ptr(out))
        return out


_cache: dict = {}


def get(kind: str = "restatement") -> Oracle:
    if kind not in _cache:
        _cache[kind] = Oracle(kind)
    return _cache[kind]


def available(kind: str) -> bool:
    return LIBS[kind].exists()


# ---------------------------------------------------------------------------
# MDR refactor / request / reconstruct of the reference library (refactor.hpp:81-117);
# only the compiled reference provides them (the C restatement does not).


class RefStore:
    """A reference RefactoredStore (opaque handle) with its manifest JSON and segment payloads."""

    def __init__(self, lib, handle):
        self.lib, self.h = lib, handle
        p = C.c_char_p()
        rc = lib.oc_mdr_manifest_json(self.h, C.byref(p))
        if rc:
            raise OracleError(rc, lib.oc_last_error().decode())
        self.manifest_json = C.string_at(p).decode()
        lib.oc_free(p)

    def segment(self, level: int, plane: int) -> bytes:
        out = P()
        n = C.c_uint64()
        rc = self.lib.oc_mdr_segment(self.h, level, plane, C.byref(out), C.byref(n))
        if rc:
            raise OracleError(rc, self.lib.oc_last_error().decode())
        b = bytes((C.c_uint8 * n.value).from_address(out.value)) if n.value else b""
        self.lib.oc_free(out)
        return b

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.oc_mdr_free(self.h)
            self.h = None


def mdr_lib():
    o = get("reference")
    L = o.lib
    L.oc_mdr_refactor.restype = P
    L.oc_mdr_refactor.argtypes = [P, C.c_int, P, P, C.c_uint32]
    L.oc_mdr_manifest_json.argtypes = [P, C.POINTER(C.c_char_p)]
    L.oc_mdr_segment.argtypes = [P, C.c_uint32, C.c_uint32, C.POINTER(P), U64P]
    L.oc_mdr_free.argtypes = [P]
    L.oc_mdr_request.argtypes = [C.c_char_p, C.c_double, C.c_int, C.c_double, P, P, P, C.c_uint64, U64P, U64P,
                                 C.POINTER(C.c_double), C.POINTER(C.c_int)]
    L.oc_mdr_session.restype = P
    L.oc_mdr_session.argtypes = [C.c_char_p, P]
    L.oc_mdr_reconstruct.argtypes = [P, P, P, C.c_uint64, C.c_int, C.c_double, P, C.POINTER(C.c_double)]
    L.oc_mdr_session_free.argtypes = [P]
    L.oc_free.argtypes = [P]
    return L


def mdr_refactor(u, planes=32, coords=None) -> RefStore:
    L = mdr_lib()
    u = np.ascontiguousarray(u, dtype=np.float64)
    shape = _shape_arr(u.shape)
    h = L.oc_mdr_refactor(_ptr(u), len(shape), _ptr(shape), _ptr(_coords_arr(coords)), planes)
    if not h:
        raise OracleError(1, L.oc_last_error().decode())
    return RefStore(L, h)


def mdr_request(manifest_json: str, tol_abs: float, norm=0, s=0.0, fetched=None):
    """-> (segments [(level, plane)], total_bytes, predicted, satisfiable) from a state with `fetched` planes."""
    L = mdr_lib()
    cap = 4096
    lv = np.zeros(cap, dtype=np.uint32)
    pl = np.zeros(cap, dtype=np.uint32)
    f = None if fetched is None else np.ascontiguousarray(fetched, dtype=np.uint32)
    n, by = C.c_uint64(), C.c_uint64()
    pred, sat = C.c_double(), C.c_int()
    rc = L.oc_mdr_request(manifest_json.encode(), tol_abs, norm, s, _ptr(f), _ptr(lv), _ptr(pl), cap, C.byref(n),
                          C.byref(by), C.byref(pred), C.byref(sat))
    if rc:
        raise OracleError(rc, L.oc_last_error().decode())
    return [(int(lv[i]), int(pl[i])) for i in range(n.value)], by.value, pred.value, bool(sat.value)


class RefSession:
    """A reference retrieval session over a RefStore (RetrievalState kept between reconstructs)."""

    def __init__(self, store: RefStore, count: int):
        self.L = mdr_lib()
        self.store = store
        self.count = count
        self.h = self.L.oc_mdr_session(store.manifest_json.encode(), store.h)
        if not self.h:
            raise OracleError(1, self.L.oc_last_error().decode())

    def reconstruct(self, segments, norm=0, s=0.0):
        lv = np.ascontiguousarray([a for a, _ in segments] or [0], dtype=np.uint32)
        pl = np.ascontiguousarray([b for _, b in segments] or [0], dtype=np.uint32)
        out = np.zeros(self.count, dtype=np.float64)
        acc = C.c_double()
        rc = self.L.oc_mdr_reconstruct(self.h, _ptr(lv), _ptr(pl), len(segments), norm, s, _ptr(out), C.byref(acc))
        if rc:
            raise OracleError(rc, self.L.oc_last_error().decode())
        return out, acc.value

    def __del__(self):
        if getattr(self, "h", None):
            self.L.oc_mdr_session_free(self.h)
            self.h = None

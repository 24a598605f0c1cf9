"""B200-native (sm_100a) MGARD-style error-bounded compression.

Python mirror of the reference's container API
(``/root/reference/proj/include/mgrc/container.hpp:66-83``) over the C-ABI in
``include/mgrc_gpu.h``.  All array work runs in the hand-written CUDA kernels
of ``csrc/``; there is no CPU fallback — without the built library or a CUDA
device every compute call raises.

    grid  = make_grid((65, 65, 65))                       # grid.cpp:56
    spec  = ErrorSpec(tol=1e-3, norm=Norm.inf, mode=Mode.rel)
    blob  = compress(u, grid, spec, Codec.huffman)        # container.hpp:69-74
    u_hat = decompress(blob)                              # container.hpp:76-77
    print(describe(inspect(blob)))                        # container.hpp:79-83

Arrays may be numpy arrays (host) or torch tensors (host or CUDA); CUDA
inputs are compressed in place without a host round trip.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import ContainerInfoC, P

__all__ = [
    "Norm", "Mode", "Codec", "DType", "ErrorSpec", "TensorGrid", "ContainerInfo", "MgrcError", "make_grid",
    "compress", "compress_to", "decompress", "decompress_into", "inspect", "describe", "plan_chunks",
    "compress_chunked", "decompress_chunked", "field_stats", "serial_sumsq", "set_device", "set_stream", "set_profiling",
    "last_profile", "launch_count", "last_compress_stats", "nlevels", "initial_bin_widths", "forward_transform",
    "inverse_transform", "quantize", "dequantize", "ERRC_NAMES",
]


class Norm(IntEnum):  # error_control.hpp:15
    inf = 0
    s = 1


class Mode(IntEnum):  # error_control.hpp:16
    abs = 0
    rel = 1


class Codec(IntEnum):  # codec.hpp:14
    raw = 0
    varint = 1
    huffman = 2


class DType(IntEnum):  # container.hpp:18
    f32 = 0
    f64 = 1


ERRC_NAMES = [
    "InvalidShape", "TooManyDims", "LevelOutOfRange", "ShapeMismatch", "NonFiniteInput", "DegenerateData",
    "Overflow", "UnknownCodec", "CorruptStream", "BadMagic", "UnsupportedVersion", "ChecksumMismatch",
    "ToleranceUnreachable", "PlaneCountOutOfRange", "UnsatisfiableTolerance", "InvalidState", "PrefixViolation",
    "BudgetTooSmall", "IoError",
]


class MgrcError(RuntimeError):
    """mgrc::error (error.hpp:34-47): ``code`` is the C-ABI status (errc ordinal + 1), ``name`` the errc name."""

    def __init__(self, code: int, message: str):
        self.code = code
        if 1 <= code <= len(ERRC_NAMES):
            self.name = ERRC_NAMES[code - 1]
        else:
            self.name = {100: "CudaError", 101: "InvalidArgument"}.get(code, f"E{code}")
        super().__init__(message)


@dataclass
class ErrorSpec:  # error_control.hpp:19-24
    tol: float = 0.0
    norm: Norm = Norm.inf
    smoothness: float = 0.0
    mode: Mode = Mode.abs


@dataclass
class TensorGrid:  # grid.hpp:15-23
    shape: tuple
    coords: Optional[list] = None

    @property
    def explicit_coords(self) -> bool:
        return self.coords is not None

    def ndims(self) -> int:
        return len(self.shape)

    def element_count(self) -> int:
        return int(np.prod(self.shape))


@dataclass
class ContainerInfo:  # container.hpp:37-51
    version: int
    constant_field: bool
    coords_present: bool
    dtype: DType
    shape: tuple
    spec: ErrorSpec
    nlevels: int
    bin_widths: list
    codec_id: int
    payload_len: int
    checksum: int
    header_size: int
    raw: bytes = field(default=b"", repr=False)
    l2_projection: bool = False  # header flag 0x04 (the L²-corrected decomposition)


def make_grid(shape: Sequence[int], coords: Optional[Sequence[Sequence[float]]] = None) -> TensorGrid:
    """make_grid (grid.cpp:56-98); validation happens in the library at compress time."""
    return TensorGrid(tuple(int(s) for s in shape), None if coords is None else [np.asarray(c, np.float64)
                                                                               for c in coords])


def _take(ptr, nbytes: int) -> memoryview:
    """A view of ``nbytes`` at a library-allocated address (ctypes.string_at takes a C int size, which
    truncates containers and arrays beyond 2 GiB)."""
    if nbytes == 0:
        return memoryview(b"")
    return memoryview((C.c_uint8 * nbytes).from_address(ptr.value if hasattr(ptr, "value") else ptr)).cast("B")


def _check(rc: int) -> None:
    if rc != 0:
        raise MgrcError(rc, _lib.lib().mgrc_gpu_last_error().decode(errors="replace"))


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _array_ptr(u):
    """(pointer, dtype code, shape, keepalive) of a numpy array or torch tensor."""
    if _is_torch(u):
        import torch

        if not u.is_contiguous():
            u = u.contiguous()
        if u.dtype == torch.float32:
            dt = DType.f32
        elif u.dtype == torch.float64:
            dt = DType.f64
        else:
            raise TypeError(f"unsupported dtype {u.dtype}")
        return u.data_ptr(), dt, tuple(u.shape), u
    a = np.asarray(u)
    if a.dtype == np.float32:
        dt = DType.f32
    elif a.dtype == np.float64:
        dt = DType.f64
    else:
        raise TypeError(f"unsupported dtype {a.dtype} (f32 or f64)")
    a = np.ascontiguousarray(a)
    return a.ctypes.data, dt, a.shape, a


def _bytes_ptr(blob):
    if _is_torch(blob):
        return blob.data_ptr(), blob.numel() * blob.element_size(), blob
    if isinstance(blob, np.ndarray):
        b = np.ascontiguousarray(blob).view(np.uint8)
        return b.ctypes.data, b.nbytes, b
    b = np.frombuffer(bytes(blob), dtype=np.uint8)
    return b.ctypes.data, b.nbytes, b


def _grid_args(grid: TensorGrid):
    shape = np.asarray(grid.shape, dtype=np.uint64)
    if grid.coords is None:
        return shape, None, []
    cs = [np.ascontiguousarray(c, dtype=np.float64) for c in grid.coords]
    arr = (P * len(cs))(*[c.ctypes.data for c in cs])
    return shape, arr, cs


def _check_grid(grid: TensorGrid, shape) -> None:
    """ShapeMismatch when the grid and the array disagree on the element count (container.cpp:76-77).

    An invalid grid shape is left to the library, which reports InvalidShape / TooManyDims first
    (make_grid validates before compress ever runs, grid.cpp:20-31) without reading the array."""
    if not (1 <= len(grid.shape) <= 4) or any(int(n) < 2 for n in grid.shape):
        return
    if int(np.prod(grid.shape, dtype=np.uint64)) != int(np.prod(shape, dtype=np.uint64)):
        raise MgrcError(4, "ShapeMismatch: array does not match the grid")


def compress(u, grid: Optional[TensorGrid] = None, spec: Optional[ErrorSpec] = None,
             codec: Codec = Codec.huffman, l2: bool = False) -> bytes:
    """mgrc::compress (container.hpp:69-74) on the GPU; returns the container bytes.
    ``l2=True``: on the decomposition with MGARD's L²-projection correction (header flag 0x04)."""
    ptr, dt, shape, keep = _array_ptr(u)
    grid = grid or make_grid(shape)
    _check_grid(grid, shape)
    spec = spec or ErrorSpec(tol=1e-3)
    gshape, coords, ckeep = _grid_args(grid)
    out = P()
    n = C.c_uint64()
    fn = _lib.lib().mgrc_gpu_compress_l2 if l2 else _lib.lib().mgrc_gpu_compress
    _check(fn(ptr, int(dt), len(gshape), gshape.ctypes.data, coords, spec.tol, int(spec.norm), spec.smoothness,
              int(spec.mode), int(codec), C.byref(out), C.byref(n)))
    b = bytes(_take(out, n.value))
    _lib.lib().mgrc_gpu_free(out)
    return b


def compress_to(u, dst, grid: Optional[TensorGrid] = None, spec: Optional[ErrorSpec] = None,
                codec: Codec = Codec.huffman, l2: bool = False) -> int:
    """Compress into a caller buffer (host numpy / torch, or a CUDA torch uint8 tensor); returns the length.

    With ``dst=None`` only the length is computed (the container stays staged on the device)."""
    ptr, dt, shape, keep = _array_ptr(u)
    grid = grid or make_grid(shape)
    _check_grid(grid, shape)
    spec = spec or ErrorSpec(tol=1e-3)
    gshape, coords, ckeep = _grid_args(grid)
    if dst is None:
        dptr, cap = None, 0
    else:
        dptr, cap, dkeep = _bytes_ptr(dst)
    n = C.c_uint64()
    fn = _lib.lib().mgrc_gpu_compress_l2_to if l2 else _lib.lib().mgrc_gpu_compress_to
    _check(fn(ptr, int(dt), len(gshape), gshape.ctypes.data, coords, spec.tol, int(spec.norm), spec.smoothness,
              int(spec.mode), int(codec), dptr, cap, C.byref(n)))
    return n.value


def decompress(blob) -> np.ndarray:
    """mgrc::decompress (container.hpp:76-77) on the GPU; returns a host numpy array."""
    ptr, n, keep = _bytes_ptr(blob)
    out = P()
    dt = C.c_int()
    nd = C.c_int()
    shape = np.zeros(4, dtype=np.uint64)
    _check(_lib.lib().mgrc_gpu_decompress(ptr, n, C.byref(out), C.byref(dt), C.byref(nd), shape.ctypes.data))
    sh = tuple(int(s) for s in shape[: nd.value])
    npdt = np.float32 if dt.value == 0 else np.float64
    cnt = int(np.prod(sh))
    arr = np.frombuffer(_take(out, cnt * np.dtype(npdt).itemsize), dtype=npdt).reshape(sh).copy()
    _lib.lib().mgrc_gpu_free(out)
    return arr


def decompress_into(blob, out) -> tuple:
    """Decompress into a caller array (numpy or torch, host or CUDA); returns (dtype, shape)."""
    ptr, n, keep = _bytes_ptr(blob)
    if _is_torch(out):
        optr, cap = out.data_ptr(), out.numel() * out.element_size()
    else:
        optr, cap = out.ctypes.data, out.nbytes
    dt = C.c_int()
    nd = C.c_int()
    shape = np.zeros(4, dtype=np.uint64)
    _check(_lib.lib().mgrc_gpu_decompress_into(ptr, n, optr, cap, C.byref(dt), C.byref(nd), shape.ctypes.data))
    return DType(dt.value), tuple(int(s) for s in shape[: nd.value])


def inspect(blob) -> ContainerInfo:
    """mgrc::inspect (container.hpp:79-80): header-only parse (host)."""
    b = bytes(blob) if not isinstance(blob, (bytes, bytearray)) else bytes(blob)
    buf = np.frombuffer(b, dtype=np.uint8)
    ci = ContainerInfoC()
    _check(_lib.lib().mgrc_gpu_inspect(buf.ctypes.data, len(b), C.byref(ci)))
    return ContainerInfo(
        version=ci.version, constant_field=bool(ci.constant_field), coords_present=bool(ci.coords_present),
        dtype=DType(ci.dtype), shape=tuple(int(ci.shape[a]) for a in range(ci.ndims)),
        spec=ErrorSpec(ci.tol, Norm(ci.norm), ci.smoothness, Mode(ci.mode)), nlevels=ci.nlevels,
        bin_widths=[ci.bin_widths[l] for l in range(ci.nlevels + 1)], codec_id=ci.codec_id,
        payload_len=ci.payload_len, checksum=ci.checksum, header_size=ci.header_size, raw=b[: ci.header_size],
        l2_projection=bool(ci.l2_projection))


def describe(info_or_blob) -> str:
    """mgrc::describe (container.hpp:82-83): stable key:value text."""
    raw = info_or_blob.raw if isinstance(info_or_blob, ContainerInfo) else bytes(info_or_blob)
    buf = np.frombuffer(raw, dtype=np.uint8)
    t = C.c_char_p()
    _check(_lib.lib().mgrc_gpu_describe(buf.ctypes.data, len(raw), C.byref(t)))
    s = t.value.decode()
    _lib.lib().mgrc_gpu_free(C.cast(t, P))
    return s


def plan_chunks(shape: Sequence[int], dtype: DType, budget: int) -> np.ndarray:
    """mgrc::plan_chunks (chunking.hpp:38-44): [nblocks, ndims, 2] ranges in block order."""
    sh = np.asarray(shape, dtype=np.uint64)
    nb = C.c_uint64()
    _check(_lib.lib().mgrc_gpu_plan_chunks(len(sh), sh.ctypes.data, int(dtype), budget, C.byref(nb), None, 0))
    out = np.zeros(int(nb.value) * len(sh) * 2, dtype=np.uint64)
    _check(_lib.lib().mgrc_gpu_plan_chunks(len(sh), sh.ctypes.data, int(dtype), budget, C.byref(nb),
                                           out.ctypes.data, nb.value))
    return out.reshape(int(nb.value), len(sh), 2)


def compress_chunked(u, spec: ErrorSpec, codec: Codec = Codec.huffman, chunk_mem: int = 0,
                     coords=None, ngpus: int = 1) -> bytes:
    """The CLI's multiblock compress (tools/mgrc.cpp:363-484) on ``ngpus`` GPUs of this process
    (mgrc_gpu_compress_chunked_multi: one host thread per GPU, NCCL all-gather of the sizes)."""
    ptr, dt, shape, keep = _array_ptr(u)
    grid = make_grid(shape, coords)
    gshape, cs, ckeep = _grid_args(grid)
    out = P()
    n = C.c_uint64()
    _check(_lib.lib().mgrc_gpu_compress_chunked_multi(ptr, int(dt), len(gshape), gshape.ctypes.data, cs, spec.tol,
                                                      int(spec.norm), spec.smoothness, int(spec.mode), int(codec),
                                                      chunk_mem, int(ngpus), C.byref(out), C.byref(n)))
    b = bytes(_take(out, n.value))
    _lib.lib().mgrc_gpu_free(out)
    return b


def decompress_chunked(blob, ngpus: int = 1) -> np.ndarray:
    """The CLI's multiblock decompress (tools/mgrc.cpp:490-542) on ``ngpus`` GPUs of this process."""
    ptr, n, keep = _bytes_ptr(blob)
    out = P()
    dt = C.c_int()
    nd = C.c_int()
    shape = np.zeros(4, dtype=np.uint64)
    _check(_lib.lib().mgrc_gpu_decompress_chunked_multi(ptr, n, int(ngpus), C.byref(out), C.byref(dt), C.byref(nd),
                                                        shape.ctypes.data))
    sh = tuple(int(s) for s in shape[: nd.value])
    npdt = np.float32 if dt.value == 0 else np.float64
    cnt = int(np.prod(sh))
    arr = np.frombuffer(_take(out, cnt * np.dtype(npdt).itemsize), dtype=npdt).reshape(sh).copy()
    _lib.lib().mgrc_gpu_free(out)
    return arr


def field_stats(u) -> tuple:
    """(min, max, nonfinite) of an array on the GPU."""
    ptr, dt, shape, keep = _array_ptr(u)
    mn = C.c_double()
    mx = C.c_double()
    nf = C.c_int()
    _check(_lib.lib().mgrc_gpu_field_stats(ptr, int(dt), int(np.prod(shape)), C.byref(mn), C.byref(mx),
                                           C.byref(nf)))
    return mn.value, mx.value, bool(nf.value)


def serial_sumsq(u, s0: float = 0.0) -> float:
    """s0 + Σ u_i² added serially in index order (the CLI's scan_stats sum, tools/mgrc.cpp:227), bit-exact,
    computed on the GPU (serial_sum.cuh)."""
    ptr, dt, shape, keep = _array_ptr(u)
    out = C.c_double()
    _check(_lib.lib().mgrc_gpu_serial_sumsq(ptr, int(dt), int(np.prod(shape)), float(s0), C.byref(out)))
    return out.value


def set_device(device: int) -> None:
    _check(_lib.lib().mgrc_gpu_set_device(device))


def set_stream(stream_handle: Optional[int]) -> None:
    """Use a caller cudaStream_t (e.g. ``torch.cuda.current_stream().cuda_stream``) on this thread."""
    _check(_lib.lib().mgrc_gpu_set_stream(stream_handle))


def set_profiling(on: bool) -> None:
    _check(_lib.lib().mgrc_gpu_set_profiling(1 if on else 0))


def launch_count() -> int:
    """Kernels launched by this thread through libmgrc_gpu.so so far."""
    return int(_lib.lib().mgrc_gpu_launch_count())


def last_profile() -> list:
    """[(phase, ms, algorithmic_bytes)] CUDA-event timings of the last call on this thread."""
    L = _lib.lib()
    out = []
    for i in range(L.mgrc_gpu_profile_count()):
        name = C.c_char_p()
        ms = C.c_double()
        by = C.c_double()
        _check(L.mgrc_gpu_profile_entry(i, C.byref(name), C.byref(ms), C.byref(by)))
        out.append((name.value.decode(), ms.value, by.value))
    return out


def last_compress_stats() -> dict:
    """Accept decision of this thread's last compress (container.cpp:93-123): ``tau_abs``, the ``achieved``
    error compared with tau_abs*(1-1e-9) (the reference's estimator; for ``decided_by == "bound"`` the
    a-priori bound (L+1)*max|r| that already passes), the shrink ``passes`` run."""
    L = _lib.lib()
    tau, ach = C.c_double(), C.c_double()
    passes, how = C.c_int(), C.c_int()
    L.mgrc_gpu_last_compress_stats(C.byref(tau), C.byref(ach), C.byref(passes), C.byref(how))
    return {"tau_abs": tau.value, "achieved": ach.value, "passes": passes.value,
            "decided_by": {0: "none", 1: "bound", 2: "exact", 3: "exact-serial"}.get(how.value, str(how.value))}


# ---------------------------------------------------------------------------
# the decomposition and the quantiser as entry points of their own
# (transform.hpp:24-30, quantize.hpp:32-42); f64 numpy arrays or torch tensors
# (host or CUDA) — outputs live where the input lives.


def _f64_ptr(a, what):
    if _is_torch(a):
        import torch

        if a.dtype != torch.float64:
            raise TypeError(f"{what} must be float64")
        a = a.contiguous()
        return a.data_ptr(), tuple(a.shape), a
    a = np.ascontiguousarray(a)
    if a.dtype != np.float64:
        raise TypeError(f"{what} must be float64")
    return a.ctypes.data, a.shape, a


def _empty_like(ref, dtype_np):
    if _is_torch(ref):
        import torch

        tdt = {np.float64: torch.float64, np.int64: torch.int64}[dtype_np]
        t = torch.empty(tuple(ref.shape), dtype=tdt, device=ref.device)
        return t, t.data_ptr()
    a = np.empty(ref.shape, dtype=dtype_np)
    return a, a.ctypes.data


def nlevels(grid: TensorGrid) -> int:
    """GridHierarchy::nlevels of the grid (grid.cpp:100-153)."""
    shape, coords, keep = _grid_args(grid)
    n = C.c_int()
    _check(_lib.lib().mgrc_gpu_nlevels(len(shape), shape.ctypes.data, coords, C.byref(n)))
    return n.value


def initial_bin_widths(tau_abs: float, spec: ErrorSpec, ndims: int, nlev: int) -> np.ndarray:
    """initial_bin_widths (error_control.cpp:42-60)."""
    out = np.zeros(nlev + 1, dtype=np.float64)
    _check(_lib.lib().mgrc_gpu_initial_bin_widths(tau_abs, int(spec.norm), spec.smoothness, ndims, nlev,
                                                  out.ctypes.data))
    return out


def forward_transform(u, grid: Optional[TensorGrid] = None, l2: bool = False):
    """forward_transform (transform.cpp:163-178) on the GPU: the multilevel coefficients of ``u``.
    ``l2=True``: with MGARD's L²-projection correction of the coarse levels (not in the reference)."""
    ptr, shape, keep = _f64_ptr(u, "u")
    grid = grid or make_grid(shape)
    _check_grid(grid, shape)
    gshape, coords, ck = _grid_args(grid)
    c, cp = _empty_like(keep, np.float64)
    fn = _lib.lib().mgrc_gpu_forward_transform_l2 if l2 else _lib.lib().mgrc_gpu_forward_transform
    _check(fn(ptr, len(gshape), gshape.ctypes.data, coords, cp))
    return c


def inverse_transform(c, grid: Optional[TensorGrid] = None, l2: bool = False):
    """inverse_transform (transform.cpp:180-191) on the GPU (``l2=True``: of the corrected decomposition)."""
    ptr, shape, keep = _f64_ptr(c, "c")
    grid = grid or make_grid(shape)
    _check_grid(grid, shape)
    gshape, coords, ck = _grid_args(grid)
    u, up = _empty_like(keep, np.float64)
    fn = _lib.lib().mgrc_gpu_inverse_transform_l2 if l2 else _lib.lib().mgrc_gpu_inverse_transform
    _check(fn(ptr, len(gshape), gshape.ctypes.data, coords, up))
    return u


def quantize(c, widths, grid: Optional[TensorGrid] = None, residuals: bool = True):
    """quantize (quantize.cpp:72-132) on the GPU: (q int64, r float64 or None, outlier count)."""
    ptr, shape, keep = _f64_ptr(c, "c")
    grid = grid or make_grid(shape)
    _check_grid(grid, shape)
    gshape, coords, ck = _grid_args(grid)
    w = np.ascontiguousarray(widths, dtype=np.float64)
    q, qp = _empty_like(keep, np.int64)
    r, rp = _empty_like(keep, np.float64) if residuals else (None, None)
    o = C.c_uint64()
    _check(_lib.lib().mgrc_gpu_quantize(ptr, len(gshape), gshape.ctypes.data, coords, w.ctypes.data, w.size, qp, rp,
                                        C.byref(o)))
    return q, r, o.value


def dequantize(q, widths, grid: Optional[TensorGrid] = None):
    """dequantize (quantize.cpp:134-158) on the GPU."""
    if _is_torch(q):
        qq = q.contiguous()
        ptr, shape = qq.data_ptr(), tuple(qq.shape)
    else:
        qq = np.ascontiguousarray(q, dtype=np.int64)
        ptr, shape = qq.ctypes.data, qq.shape
    grid = grid or make_grid(shape)
    _check_grid(grid, shape)
    gshape, coords, ck = _grid_args(grid)
    w = np.ascontiguousarray(widths, dtype=np.float64)
    if _is_torch(q):
        import torch

        c = torch.empty(shape, dtype=torch.float64, device=q.device)
        cp = c.data_ptr()
    else:
        c = np.empty(shape, dtype=np.float64)
        cp = c.ctypes.data
    _check(_lib.lib().mgrc_gpu_dequantize(ptr, len(gshape), gshape.ctypes.data, coords, w.ctypes.data, w.size, cp))
    return c

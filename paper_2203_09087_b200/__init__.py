"""paper_2203_09087_b200 -- B200-native Euler characteristic curves.

Python binding of the C ABI in ``include/ecc_b200.h`` (the product is the
CUDA library ``lib/libecc_b200.so``; C++ callers use the drop-in headers in
``include/ecc/``).  Names mirror the reference API in
``/root/reference/proj/include/ecc`` so tests read like the reference's own:

=====================================  =========================================
reference (file:line)                  here
=====================================  =========================================
``Dims`` (common.hpp:18-31)            :class:`Dims`
``ChunkRange/ChunkPlan/ChunkTarget``   :class:`ChunkRange`, :class:`ChunkPlan`,
(streaming.hpp:21-46)                  :class:`ChunkTarget`
``plan_chunks`` (streaming.hpp:65-81)  :func:`plan_chunks`
``process_image`` (streaming.hpp:      :func:`process_image` (array, device
181-338)                               tensor, or :class:`ChunkSource`)
``GlobalVcec`` (vcec.hpp:15-31)        :class:`GlobalVcec`
``vcec_to_ecc`` (curve.hpp:28-35)      :func:`vcec_to_ecc`
``compute_changes`` (kernel.hpp:       :func:`compute_changes`
244-265)
(new) batched 2D                       :func:`batch2d`
=====================================  =========================================

There is no CPU fallback: every call goes through the CUDA library and fails
loudly (:class:`EccError`) when it or the GPU is missing.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
import threading
import weakref
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# ECC_B200_LIB: load another build of the same library (variant experiments)
LIB_PATH = os.environ.get("ECC_B200_LIB") or os.path.join(PKG, "lib", "libecc_b200.so")

ECC_OK, ECC_EINVAL, ECC_ECUDA, ECC_ENOMEM, ECC_ESOURCE, ECC_EBINMAP, ECC_ENAN = 0, -1, -2, -3, -4, -5, -6
ECC_U8, ECC_U16, ECC_F32 = 0, 1, 2
ECC_BIN_IDENTITY, ECC_BIN_AFFINE, ECC_BIN_SORTED = 0, 1, 2


class EccError(RuntimeError):
    """ecc::error (common.hpp:11-14) carried across the C ABI."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class _Dims(C.Structure):
    _fields_ = [("w0", C.c_uint64), ("w1", C.c_uint64), ("w2", C.c_uint64)]


class _BinMap(C.Structure):
    _fields_ = [("kind", C.c_int32), ("nbins", C.c_uint32), ("lo", C.c_float), ("step", C.c_float)]


class _Timing(C.Structure):
    _fields_ = [("begin", C.c_uint64), ("end", C.c_uint64),
                ("ingest_begin", C.c_double), ("ingest_end", C.c_double),
                ("index_begin", C.c_double), ("index_end", C.c_double),
                ("kernel_begin", C.c_double), ("kernel_end", C.c_double),
                ("merge_begin", C.c_double), ("merge_end", C.c_double)]


class _BenchReport(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("voxels", C.c_uint64),
                ("generate_s", C.c_double), ("total_s", C.c_double),
                ("per_iteration_s", C.c_double), ("ecc_avg_s", C.c_double),
                ("smooth_avg_s", C.c_double), ("ecc_gvox_per_s", C.c_double),
                ("last_points", C.c_uint64), ("last_chi_first", C.c_int64),
                ("last_chi_last", C.c_int64)]


READ_ROWS_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                           C.c_void_p, C.c_size_t)

_lib = None
_lib_lock = threading.Lock()
_vp, _u64, _i64 = C.c_void_p, C.c_uint64, C.c_int64


def lib() -> C.CDLL:
    """Loads the CUDA library; raises if it has not been built."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise EccError(ECC_ECUDA, f"CUDA library missing: {LIB_PATH} (run __graft_entry__.build())")
            L = C.CDLL(LIB_PATH)
            L.ecc_last_error.restype = C.c_char_p
            L.ecc_abi_version.restype = C.c_int
            L.ecc_ctx_create.argtypes = [C.c_int, C.POINTER(_vp)]
            L.ecc_ctx_destroy.argtypes = [_vp]
            L.ecc_ctx_destroy.restype = None
            L.ecc_ctx_stream.argtypes = [_vp]
            L.ecc_ctx_stream.restype = _vp
            L.ecc_ctx_launch_count.argtypes = [_vp]
            L.ecc_ctx_launch_count.restype = _u64
            L.ecc_bin_count.argtypes = [C.c_int, C.POINTER(_BinMap), C.POINTER(_u64)]
            slab = [_vp, _vp, C.c_int, _Dims, _u64, _u64, _u64, _u64]
            L.ecc_accumulate_slab.argtypes = slab + [C.POINTER(_BinMap), _vp, _vp]
            L.ecc_compute_changes.argtypes = slab + [_vp, _vp]
            L.ecc_finalize.argtypes = [_vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp]
            L.ecc_process_host.argtypes = [_vp, _vp, C.c_int, _Dims, C.POINTER(_u64), C.c_size_t,
                                           C.POINTER(_BinMap), C.POINTER(_Timing), _vp, _vp, _u64,
                                           C.POINTER(_u64)]
            L.ecc_accumulate_host.argtypes = [_vp, _vp, _u64, _u64, C.c_int, _Dims,
                                              C.POINTER(_u64), C.c_size_t, C.POINTER(_BinMap), _vp]
            L.ecc_accumulate_host.restype = C.c_int
            L.ecc_batch_format.argtypes = [_vp, _vp, _vp, _u64, C.c_int, C.c_int, _vp, _u64,
                                           _vp, C.POINTER(_u64)]
            L.ecc_batch_format.restype = C.c_int
            L.ecc_format_curve.argtypes = [_vp, C.c_int, _vp, _vp, _u64, C.c_int, C.c_int, _vp, _u64,
                                           C.POINTER(_u64)]
            L.ecc_format_curve.restype = C.c_int
            L.ecc_batch_zero_crossings.argtypes = [_vp, _vp, _vp, _u64, C.c_int, _vp, _vp]
            L.ecc_batch_zero_crossings.restype = C.c_int
            L.ecc_xchg_create.argtypes = [_vp, C.c_int, C.c_int, C.POINTER(_vp), _vp]
            L.ecc_xchg_create.restype = C.c_int
            L.ecc_xchg_open.argtypes = [_vp, _vp]
            L.ecc_xchg_open.restype = C.c_int
            L.ecc_xchg_destroy.argtypes = [_vp]
            L.ecc_xchg_destroy.restype = None
            L.ecc_xchg_status.argtypes = [_vp]
            L.ecc_xchg_status.restype = C.c_int
            L.ecc_curve_sharded.argtypes = [_vp, _vp, _vp, _Dims, _u64, _u64, _u64, _u64,
                                            _vp, _vp, _vp, _vp, _vp]
            L.ecc_curve_sharded.restype = C.c_int
            L.ecc_process_file.argtypes = [_vp, C.c_char_p, C.c_int, _Dims, C.c_int, C.POINTER(_u64),
                                           C.c_size_t, C.POINTER(_BinMap), C.POINTER(_Timing), _vp,
                                           _vp, _u64, C.POINTER(_u64)]
            L.ecc_curve_device.argtypes = [_vp, _vp, C.c_int, _Dims, C.POINTER(_BinMap), _vp, _vp,
                                           _vp, _vp, _vp]
            vol = [_vp, _vp, C.c_int, C.c_int, _Dims, C.POINTER(_BinMap), _vp, _vp, _u64, C.POINTER(_u64)]
            L.ecc_vcec.argtypes = vol
            L.ecc_curve.argtypes = vol
            L.ecc_process_stream.argtypes = [_vp, READ_ROWS_FN, _vp, C.c_int, _Dims, C.POINTER(_u64),
                                             C.c_size_t, C.POINTER(_BinMap), C.POINTER(_Timing),
                                             _vp, _vp, _u64, C.POINTER(_u64)]
            L.ecc_batch2d.argtypes = [_vp, _vp, C.c_int, C.c_int, _u64, _u64, _u64, _vp, _vp, _vp]
            L.ecc_fill_synthetic.argtypes = [_vp, _vp, C.c_int, _u64, _u64, _u64, _vp]
            L.ecc_uniform_noise.argtypes = [_vp, _vp, _u64, _u64, _vp]
            L.ecc_gaussian_smooth.argtypes = [_vp, _vp, _vp, _Dims, C.c_double, C.c_int, _vp]
            L.ecc_bench_run.argtypes = [_vp, _Dims, _u64, _u64, C.c_double, C.c_int,
                                        C.POINTER(_BenchReport)]
            for n in ("ecc_ctx_create", "ecc_bin_count", "ecc_accumulate_slab", "ecc_compute_changes",
                      "ecc_finalize", "ecc_vcec", "ecc_curve", "ecc_process_stream", "ecc_batch2d",
                      "ecc_fill_synthetic", "ecc_curve_device", "ecc_process_host",
                      "ecc_process_file", "ecc_uniform_noise", "ecc_gaussian_smooth",
                      "ecc_bench_run"):
                getattr(L, n).restype = C.c_int
            _lib = L
        return _lib


def _check(rc: int):
    if rc != ECC_OK:
        raise EccError(rc, lib().ecc_last_error().decode(errors="replace"))


# ------------------------------------------------------------------ types
@dataclass(frozen=True)
class Dims:
    """Grid dims; axis 0 slowest, 2D images have w2 == 1 (common.hpp:18-31)."""
    w0: int = 1
    w1: int = 1
    w2: int = 1

    def voxel_count(self) -> int:
        return self.w0 * self.w1 * self.w2

    def is_2d(self) -> bool:
        return self.w2 == 1

    def to_string(self) -> str:
        return f"{self.w0}x{self.w1}x{self.w2}"

    @staticmethod
    def of(shape) -> "Dims":
        if len(shape) == 2:
            return Dims(int(shape[0]), int(shape[1]), 1)
        if len(shape) == 3:
            return Dims(int(shape[0]), int(shape[1]), int(shape[2]))
        raise EccError(ECC_EINVAL, f"expected a 2D or 3D image, got shape {tuple(shape)}")


@dataclass(frozen=True)
class ChunkRange:
    begin: int = 0
    end: int = 0

    def len(self) -> int:
        return self.end - self.begin


@dataclass
class ChunkPlan:
    ranges: List[ChunkRange] = field(default_factory=list)

    def chunk_count(self) -> int:
        return len(self.ranges)


@dataclass
class ChunkTarget:
    chunks: Optional[int] = None
    budget_bytes: Optional[int] = None

    @staticmethod
    def count(c: int) -> "ChunkTarget":
        return ChunkTarget(chunks=c)

    @staticmethod
    def memory_budget(b: int) -> "ChunkTarget":
        return ChunkTarget(budget_bytes=b)


def _even_plan(w0: int, c: int) -> ChunkPlan:
    """even_plan (streaming.hpp:50-58): ceiling lengths, last chunk absorbs."""
    c = max(1, min(c, w0))
    ln = (w0 + c - 1) // c
    return ChunkPlan([ChunkRange(a, min(a + ln, w0)) for a in range(0, w0, ln)])


_EXT_BYTES = {np.dtype(np.uint8): 2, np.dtype(np.uint16): 4, np.dtype(np.float32): 4}


def padded_chunk_bytes(dims: Dims, length: int, dtype=np.float32) -> int:
    """padded_chunk_bytes (chunk.hpp:40-44) in the reference's extended type."""
    return (length + 2) * (dims.w1 + 2) * (dims.w2 + 2) * _EXT_BYTES[np.dtype(dtype)]


def plan_chunks(dims: Dims, target: ChunkTarget, dtype=np.float32) -> ChunkPlan:
    """plan_chunks (streaming.hpp:65-81), same messages."""
    if dims.w0 < 1:
        raise EccError(ECC_EINVAL, "w0 must be >= 1")
    if target.chunks is not None:
        return _even_plan(dims.w0, target.chunks)
    if target.budget_bytes is None:
        raise EccError(ECC_EINVAL, "chunk target needs a count or a memory budget")
    slab = padded_chunk_bytes(dims, 1, dtype) // 3
    minimum = 2 * padded_chunk_bytes(dims, 1, dtype)
    if target.budget_bytes < minimum:
        raise EccError(ECC_EINVAL, f"memory budget {target.budget_bytes} bytes is below the minimum "
                                   f"feasible {minimum} bytes (two single-row padded chunks)")
    ln = target.budget_bytes // (2 * slab) - 2
    c = (dims.w0 + ln - 1) // ln
    return _even_plan(dims.w0, c)


@dataclass
class GlobalVcec:
    """GlobalVcec (vcec.hpp:15-31): ascending occurring values + int64 changes."""
    values: np.ndarray
    changes: np.ndarray

    def size(self) -> int:
        return len(self.values)

    def total(self) -> int:
        return int(self.changes.sum())

    def change_for(self, v) -> int:
        i = np.searchsorted(self.values, v)
        if i < len(self.values) and self.values[i] == v:
            return int(self.changes[i])
        return 0


@dataclass
class EccCurve:
    """EccCurve (curve.hpp:18-25)."""
    thresholds: np.ndarray
    chi: np.ndarray

    def size(self) -> int:
        return len(self.thresholds)

    def __eq__(self, other) -> bool:
        return (np.array_equal(self.thresholds, other.thresholds)
                and np.array_equal(self.chi, other.chi))


def vcec_to_ecc(vcec: GlobalVcec) -> EccCurve:
    """vcec_to_ecc (curve.hpp:28-35): int64 prefix sum."""
    if vcec.size() == 0:
        raise EccError(ECC_EINVAL, "cannot build an ECC from an empty VCEC")
    return EccCurve(vcec.values.copy(), np.cumsum(vcec.changes, dtype=np.int64))


@dataclass
class ChunkTiming:
    range: ChunkRange
    ingest_begin: float = 0.0
    ingest_end: float = 0.0
    index_begin: float = 0.0
    index_end: float = 0.0
    kernel_begin: float = 0.0
    kernel_end: float = 0.0
    merge_begin: float = 0.0
    merge_end: float = 0.0


@dataclass
class EngineReport:
    chunks: List[ChunkTiming] = field(default_factory=list)
    read_s: float = 0.0
    index_s: float = 0.0
    kernel_s: float = 0.0
    merge_s: float = 0.0
    peak_chunk_bytes: int = 0


@dataclass
class BenchReport:
    """BenchReport (pipeline.hpp:212-233) of the GPU-resident bench_run, plus
    the last iteration's curve summary."""
    iterations: int = 0
    voxels: int = 0
    generate_s: float = 0.0
    total_s: float = 0.0
    per_iteration_s: float = 0.0
    ecc_avg_s: float = 0.0
    smooth_avg_s: float = 0.0
    ecc_gvox_per_s: float = 0.0
    last_points: int = 0
    last_chi_first: int = 0
    last_chi_last: int = 0

    def to_string(self) -> str:
        """Same lines as the reference's BenchReport::to_string."""
        return (f"iterations:       {self.iterations}\n"
                f"voxels:           {self.voxels}\n"
                f"generate:         {self.generate_s:g} s\n"
                f"loop total:       {self.total_s:g} s\n"
                f"per iteration:    {self.per_iteration_s:g} s\n"
                f"ECC avg:          {self.ecc_avg_s:g} s\n"
                f"smoothing avg:    {self.smooth_avg_s:g} s\n"
                f"ECC GVox/s:       {self.ecc_gvox_per_s:g}\n")


@dataclass
class EngineOptions:
    workers: int = 1           # accepted for API parity; the GPU ignores it
    ingest_delay_ms: float = 0.0  # test hook (streaming.hpp:97-101)
    device: int = 0


class ChunkSource:
    """ChunkSource (chunk.hpp:131-137): read_rows fills dst with rows [r0, r1)."""

    def dims(self) -> Dims:
        raise NotImplementedError

    def dtype(self):
        raise NotImplementedError

    def read_rows(self, r0: int, r1: int, dst: np.ndarray) -> None:
        raise NotImplementedError


class MemorySource(ChunkSource):
    """MemorySource (chunk.hpp:139-152) over a host array."""

    def __init__(self, image: np.ndarray):
        self._img = np.ascontiguousarray(image)
        self._dims = Dims.of(self._img.shape)

    def dims(self) -> Dims:
        return self._dims

    def dtype(self):
        return self._img.dtype

    def read_rows(self, r0, r1, dst):
        row = self._dims.w1 * self._dims.w2
        dst[:] = self._img.reshape(-1)[r0 * row:r1 * row]


# ------------------------------------------------------------------ context
_DT = {np.dtype(np.uint8): ECC_U8, np.dtype(np.uint16): ECC_U16, np.dtype(np.float32): ECC_F32}
_NP = {ECC_U8: np.uint8, ECC_U16: np.uint16, ECC_F32: np.float32}


def _binmap(dtype_code: int, binmap) -> Optional[_BinMap]:
    if binmap is None:
        if dtype_code == ECC_F32:
            return _BinMap(ECC_BIN_SORTED, 0, 0.0, 0.0)
        return _BinMap(ECC_BIN_IDENTITY, 0, 0.0, 0.0)
    if isinstance(binmap, _BinMap):
        return binmap
    kind = binmap.get("kind", "affine")
    if kind == "affine":
        return _BinMap(ECC_BIN_AFFINE, int(binmap["nbins"]), float(binmap.get("lo", 0.0)),
                       float(binmap["step"]))
    if kind == "sorted":
        return _BinMap(ECC_BIN_SORTED, 0, 0.0, 0.0)
    if kind == "identity":
        return _BinMap(ECC_BIN_IDENTITY, 0, 0.0, 0.0)
    raise EccError(ECC_EINVAL, f"unknown bin map {kind!r}")


def quantised_binmap(levels: int = 65536, lo: float = 0.0, hi: float = 1.0) -> dict:
    """Affine grid lo + k*(hi-lo)/levels, e.g. BASELINE config 4 (k * 2^-16)."""
    return {"kind": "affine", "nbins": levels, "lo": lo, "step": (hi - lo) / levels}


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


_live = weakref.WeakSet()


_CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy


class Context:
    """One ecc_ctx (one GPU, its streams and scratch)."""

    def __init__(self, device: int = 0):
        self._p = _vp()
        _check(lib().ecc_ctx_create(int(device), C.byref(self._p)))
        self.device = device
        _live.add(self)

    def _s(self, stream):
        """The CUDA stream a device-tensor call runs on: the caller's, else
        torch's current stream on this device, so the call is ordered with
        the torch work that produced / consumes its tensors."""
        if stream:
            return stream
        import torch
        h = torch.cuda.current_stream(self.device).cuda_stream
        # torch's default stream has handle 0, which the C ABI reads as "the
        # context's stream": name the legacy default stream explicitly
        return h if h else _CUDA_STREAM_LEGACY

    def close(self):
        if self._p:
            lib().ecc_ctx_destroy(self._p)
            self._p = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return lib().ecc_ctx_stream(self._p) or 0

    def launch_count(self) -> int:
        return int(lib().ecc_ctx_launch_count(self._p))

    # -------------------------------------------------------------- whole volume
    def _volume(self, fn, image, binmap, stream_to_sync=None):
        if _is_torch_cuda(image):
            import torch
            dt = {torch.uint8: ECC_U8, torch.uint16: ECC_U16, torch.float32: ECC_F32}[image.dtype]
            image = image.contiguous()
            dims = Dims.of(tuple(image.shape))
            data, where = image.data_ptr(), 1
            torch.cuda.current_stream(image.device).synchronize()
        else:
            image = np.ascontiguousarray(image)
            dt = _DT[image.dtype]
            dims = Dims.of(image.shape)
            data, where = image.ctypes.data, 0
        bm = _binmap(dt, binmap)
        cap = 256 if dt == ECC_U8 else (65536 if dt == ECC_U16 else dims.voxel_count())
        if dt == ECC_F32 and bm.kind == ECC_BIN_AFFINE:
            cap = bm.nbins
        elif dt == ECC_F32:
            # distinct f32 values: rarely near one per voxel, so start at 4 M
            # points (48 MB) and call again at the exact size if they are more
            cap = min(cap, 1 << 22)

        def run(cap):
            vals = np.empty(cap, _NP[dt])
            series = np.empty(cap, np.int64)
            n = _u64()
            rc = fn(self._p, data, where, dt, _Dims(dims.w0, dims.w1, dims.w2), C.byref(bm),
                    vals.ctypes.data, series.ctypes.data, cap, C.byref(n))
            return rc, vals, series, n.value

        rc, vals, series, m = run(cap)
        if rc == ECC_EINVAL and m > cap:  # "output capacity ... is below the m values"
            rc, vals, series, m = run(m)
        _check(rc)
        if 2 * m < cap:  # small result: do not keep the oversized arrays alive
            return vals[:m].copy(), series[:m].copy()
        return vals[:m], series[:m]

    def vcec(self, image, binmap=None) -> GlobalVcec:
        v, c = self._volume(lib().ecc_vcec, image, binmap)
        return GlobalVcec(v, c)

    def curve(self, image, binmap=None) -> EccCurve:
        t, chi = self._volume(lib().ecc_curve, image, binmap)
        return EccCurve(t, chi)

    # -------------------------------------------------------------- streaming
    def process_host(self, image, plan: ChunkPlan, report: EngineReport = None,
                     binmap=None) -> GlobalVcec:
        """process_image over a plan for a host array (ecc_process_host):
        each chunk + halo rows is DMA-copied straight from `image` (page-locked
        memory -- e.g. a pinned torch tensor's .numpy() -- streams at full
        PCIe speed) while the previous chunks' kernels run."""
        if not isinstance(image, np.ndarray):
            image = image.numpy()
        image = np.ascontiguousarray(image)
        dt = _DT[image.dtype]
        np_t = _NP[dt]
        dims = Dims.of(image.shape)
        ranges = plan.ranges
        bounds = (_u64 * (len(ranges) + 1))()
        if ranges:
            bounds[0] = ranges[0].begin
            for k, r in enumerate(ranges):
                bounds[k + 1] = r.end
                if k > 0 and r.begin != ranges[k - 1].end:
                    raise EccError(ECC_EINVAL, "chunk plan does not cover the image contiguously")
        bm = _binmap(dt, binmap)
        cap = 256 if dt == ECC_U8 else (65536 if dt == ECC_U16 else max(1, bm.nbins))
        vals = np.empty(cap, np_t)
        ch = np.empty(cap, np.int64)
        tim = (_Timing * max(1, len(ranges)))()
        n = _u64()
        _check(lib().ecc_process_host(self._p, image.ctypes.data, dt, _Dims(dims.w0, dims.w1, dims.w2),
                                      bounds, len(ranges), C.byref(bm), tim, vals.ctypes.data,
                                      ch.ctypes.data, cap, C.byref(n)))
        if report is not None:
            report.chunks = [ChunkTiming(ChunkRange(t.begin, t.end), t.ingest_begin, t.ingest_end,
                                         t.index_begin, t.index_end, t.kernel_begin, t.kernel_end,
                                         t.merge_begin, t.merge_end) for t in tim[:len(ranges)]]
        m = n.value
        return GlobalVcec(vals[:m].copy(), ch[:m].copy())

    def process_file(self, path: str, dims: Dims, dtype, plan: ChunkPlan = None,
                     big_endian: bool = False, binmap=None,
                     report: EngineReport = None) -> GlobalVcec:
        """process_image over the reference's FileSource (chunk.hpp:154-189):
        raw row-major file, chunked pread into pinned staging; f32 byte swap
        and NaN rejection run on the GPU (ecc_process_file)."""
        dt = _DT[np.dtype(dtype)]
        np_t = _NP[dt]
        plan = plan or _even_plan(dims.w0, 1)
        ranges = plan.ranges
        bounds = (_u64 * (len(ranges) + 1))()
        if ranges:
            bounds[0] = ranges[0].begin
            for k, r in enumerate(ranges):
                bounds[k + 1] = r.end
        bm = _binmap(dt, binmap)
        cap = 256 if dt == ECC_U8 else (65536 if dt == ECC_U16 else
                                         (bm.nbins if bm.kind == ECC_BIN_AFFINE else dims.voxel_count()))
        vals = np.empty(max(1, cap), np_t)
        ch = np.empty(max(1, cap), np.int64)
        tim = (_Timing * max(1, len(ranges)))()
        n = _u64()
        _check(lib().ecc_process_file(self._p, os.fsencode(path), dt, _Dims(dims.w0, dims.w1, dims.w2),
                                      int(big_endian), bounds, len(ranges), C.byref(bm), tim,
                                      vals.ctypes.data, ch.ctypes.data, cap, C.byref(n)))
        if report is not None:
            report.chunks = [ChunkTiming(ChunkRange(t.begin, t.end), t.ingest_begin, t.ingest_end,
                                         t.index_begin, t.index_end, t.kernel_begin, t.kernel_end,
                                         t.merge_begin, t.merge_end) for t in tim[:len(ranges)]]
        m = n.value
        return GlobalVcec(vals[:m].copy(), ch[:m].copy())

    def process_source(self, source: ChunkSource, plan: ChunkPlan, options: EngineOptions = None,
                       report: EngineReport = None, binmap=None) -> GlobalVcec:
        """process_image(ChunkSource&, plan) (streaming.hpp:181-329)."""
        options = options or EngineOptions()
        dims = source.dims()
        dt = _DT[np.dtype(source.dtype())]
        np_t = _NP[dt]
        row = dims.w1 * dims.w2
        err_holder = []
        import time as _time

        def cb(user, r0, r1, dst, errbuf, errlen):
            try:
                if options.ingest_delay_ms > 0:
                    _time.sleep(options.ingest_delay_ms / 1000.0)
                n = (r1 - r0) * row
                buf = np.ctypeslib.as_array(C.cast(dst, C.POINTER(np.ctypeslib.as_ctypes_type(np_t))),
                                            shape=(n,))
                source.read_rows(int(r0), int(r1), buf)
                return 0
            except Exception as e:  # propagate the message like streaming.hpp:250-259
                msg = str(e).encode()[: errlen - 1]
                C.memmove(errbuf, msg, len(msg))
                err_holder.append(e)
                return 1

        fn = READ_ROWS_FN(cb)
        ranges = plan.ranges
        bounds = (_u64 * (len(ranges) + 1))()
        if ranges:
            bounds[0] = ranges[0].begin
            for k, r in enumerate(ranges):
                bounds[k + 1] = r.end
                if k > 0 and r.begin != ranges[k - 1].end:
                    raise EccError(ECC_EINVAL, "chunk plan does not cover the image contiguously")
        bm = _binmap(dt, binmap)
        cap = 256 if dt == ECC_U8 else (65536 if dt == ECC_U16 else dims.voxel_count())
        if dt == ECC_F32 and bm.kind == ECC_BIN_AFFINE:
            cap = bm.nbins
        vals = np.empty(cap, np_t)
        ch = np.empty(cap, np.int64)
        tim = (_Timing * max(1, len(ranges)))()
        n = _u64()
        _check(lib().ecc_process_stream(self._p, fn, None, dt, _Dims(dims.w0, dims.w1, dims.w2),
                                        bounds, len(ranges), C.byref(bm), tim, vals.ctypes.data,
                                        ch.ctypes.data, cap, C.byref(n)))
        if report is not None:
            report.chunks = []
            for k in range(len(ranges)):
                t = tim[k]
                report.chunks.append(ChunkTiming(ChunkRange(t.begin, t.end), t.ingest_begin,
                                                 t.ingest_end, t.index_begin, t.index_end,
                                                 t.kernel_begin, t.kernel_end, t.merge_begin,
                                                 t.merge_end))
            report.read_s = sum(c.ingest_end - c.ingest_begin for c in report.chunks)
            report.kernel_s = sum(c.kernel_end - c.kernel_begin for c in report.chunks)
            report.merge_s = sum(c.merge_end - c.merge_begin for c in report.chunks)
            maxlen = max(r.len() for r in ranges)
            report.peak_chunk_bytes = 2 * (maxlen + 2) * row * np.dtype(np_t).itemsize
        m = n.value
        return GlobalVcec(vals[:m].copy(), ch[:m].copy())

    # -------------------------------------------------------------- lower level
    def accumulate_host(self, planes, plane0: int, dims: Dims, bounds, hist, binmap=None):
        """ecc_accumulate_host: a rank's owned planes [bounds[0], bounds[-1])
        of a host image whose planes [plane0, plane0 + len(planes)) are in
        `planes` (numpy or a CPU torch tensor; pinned memory streams at full
        PCIe speed), accumulated chunk by chunk into the device int64
        histogram `hist` (torch, 2*nbins, not zeroed here)."""
        import torch
        if not isinstance(planes, np.ndarray):
            planes = planes.numpy()
        planes = np.ascontiguousarray(planes)
        dt = _DT[planes.dtype]
        b = (_u64 * len(bounds))(*[int(x) for x in bounds])
        # the call runs on the context's streams and returns when done: the
        # torch work that produced `hist` (e.g. its zero-fill) must be done
        torch.cuda.current_stream(self.device).synchronize()
        bm = _binmap(dt, binmap)
        _check(lib().ecc_accumulate_host(self._p, planes.ctypes.data, plane0, planes.shape[0], dt,
                                         _Dims(dims.w0, dims.w1, dims.w2), b, len(bounds) - 1,
                                         C.byref(bm), hist.data_ptr()))

    def accumulate_slab(self, planes, dims: Dims, plane0: int, own0: int, own1: int,
                        hist, binmap=None, stream: int = 0):
        """K1+K2 into a device int64 histogram tensor of 2*nbins (torch)."""
        import torch
        dt = {torch.uint8: ECC_U8, torch.uint16: ECC_U16, torch.float32: ECC_F32}[planes.dtype]
        nplanes = planes.numel() // (dims.w1 * dims.w2)
        bm = _binmap(dt, binmap)
        _check(lib().ecc_accumulate_slab(self._p, planes.data_ptr(), dt,
                                         _Dims(dims.w0, dims.w1, dims.w2), plane0, nplanes, own0,
                                         own1, C.byref(bm), hist.data_ptr(), self._s(stream)))

    def compute_changes(self, planes, dims: Dims, plane0: int, own0: int, own1: int, out,
                        stream: int = 0):
        import torch
        dt = {torch.uint8: ECC_U8, torch.uint16: ECC_U16, torch.float32: ECC_F32}[planes.dtype]
        nplanes = planes.numel() // (dims.w1 * dims.w2)
        _check(lib().ecc_compute_changes(self._p, planes.data_ptr(), dt,
                                         _Dims(dims.w0, dims.w1, dims.w2), plane0, nplanes, own0,
                                         own1, out.data_ptr(), self._s(stream)))

    def curve_device(self, image, dims: Dims, bins, changes, chi, count, binmap=None,
                     stream: int = 0):
        """Device-resident image -> curve in device tensors (ecc_curve_device):
        one fused launch for 3D u8 volumes."""
        import torch
        dt = {torch.uint8: ECC_U8, torch.uint16: ECC_U16, torch.float32: ECC_F32}[image.dtype]
        bm = _binmap(dt, binmap)
        _check(lib().ecc_curve_device(self._p, image.data_ptr(), dt, _Dims(dims.w0, dims.w1, dims.w2),
                                      C.byref(bm), bins.data_ptr(), changes.data_ptr(),
                                      chi.data_ptr(), count.data_ptr(), self._s(stream)))

    def curve_sharded(self, xchg: "Exchange", planes, dims: Dims, plane0: int, own0: int,
                      own1: int, bins, changes, chi, count, stream: int = 0):
        """ecc_curve_sharded: this rank's slab -> the GLOBAL curve on every
        rank, the histogram exchange fused into the launch (see Exchange)."""
        nplanes = planes.numel() // (dims.w1 * dims.w2)
        _check(lib().ecc_curve_sharded(self._p, xchg._p, planes.data_ptr(),
                                       _Dims(dims.w0, dims.w1, dims.w2), plane0, nplanes, own0,
                                       own1, bins.data_ptr(), changes.data_ptr(), chi.data_ptr(),
                                       count.data_ptr(), self._s(stream)))

    def finalize(self, hist, nbins: int, bins, changes, chi, count, stream: int = 0):
        _check(lib().ecc_finalize(self._p, hist.data_ptr(), nbins, bins.data_ptr(),
                                  changes.data_ptr(), chi.data_ptr(), count.data_ptr(),
                                  self._s(stream)))

    def batch2d(self, images, chi=None, presence=None, stream: int = 0):
        """Dense per-image curves for a (count, h, w) stack: chi (count, nbins)
        int32 and presence bitmaps (count, nbins/32) uint32."""
        if _is_torch_cuda(images):
            import torch
            dt = {torch.uint8: ECC_U8, torch.uint16: ECC_U16}[images.dtype]
            count, h, w = images.shape
            nb = 256 if dt == ECC_U8 else 65536
            if chi is None:
                chi = torch.empty((count, nb), dtype=torch.int32, device=images.device)
            if presence is None:
                presence = torch.empty((count, nb // 32), dtype=torch.int32, device=images.device)
            _check(lib().ecc_batch2d(self._p, images.data_ptr(), 1, dt, count, h, w,
                                     chi.data_ptr(), presence.data_ptr(), self._s(stream)))
            return chi, presence
        images = np.ascontiguousarray(images)
        dt = _DT[images.dtype]
        count, h, w = images.shape
        nb = 256 if dt == ECC_U8 else 65536
        chi = np.empty((count, nb), np.int32)
        presence = np.empty((count, nb // 32), np.uint32)
        _check(lib().ecc_batch2d(self._p, images.ctypes.data, 0, dt, count, h, w,
                                 chi.ctypes.data, presence.ctypes.data, None))
        return chi, presence

    def uniform_noise(self, tensor, seed: int = 0, stream: int = 0):
        """uniform_noise (datagen.hpp:57-62) into a device float32 tensor."""
        _check(lib().ecc_uniform_noise(self._p, tensor.data_ptr(), tensor.numel(), seed,
                                       self._s(stream)))
        return tensor

    def gaussian_smooth(self, tensor, sigma: float, width: int, out=None, stream: int = 0):
        """gaussian_smooth (datagen.hpp:108-122) of a device float32 tensor
        (2D or 3D), bit-identical to the reference; out may be the input."""
        import torch
        if out is None:
            out = torch.empty_like(tensor)
        _check(lib().ecc_gaussian_smooth(self._p, tensor.data_ptr(), out.data_ptr(),
                                         _dims_of(tuple(tensor.shape)), sigma, width,
                                         self._s(stream)))
        return out

    def bench_run(self, dims: Dims, iterations: int, seed: int = 1, sigma: float = 2.0,
                  width: int = 13) -> BenchReport:
        """bench_run (pipeline.hpp:236-291) on the GPU: uniform noise once, then
        `iterations` x {gaussian_smooth; ECC on the exact f32 path}, all in
        device memory."""
        r = _BenchReport()
        _check(lib().ecc_bench_run(self._p, _Dims(dims.w0, dims.w1, dims.w2), iterations, seed,
                                   sigma, width, C.byref(r)))
        return BenchReport(**{f: getattr(r, f) for f, _ in _BenchReport._fields_})

    def batch_format(self, chi, presence, dtype=np.uint16, fmt: str = "csv"):
        """write_curve bytes (curve.hpp:87-121) of every image of a device
        batch (batch2d's chi / presence tensors), formatted on the GPU:
        returns one bytes object per image."""
        dt = _DT[np.dtype(dtype)]
        count = chi.shape[0]
        f = {"csv": 0, "json": 1}[fmt]
        offs = np.empty(count + 1, np.uint64)
        total = _u64()
        _check(lib().ecc_batch_format(self._p, chi.data_ptr(), presence.data_ptr(), count, dt, f,
                                      None, 0, offs.ctypes.data, C.byref(total)))
        out = np.empty(max(1, total.value), np.uint8)
        _check(lib().ecc_batch_format(self._p, chi.data_ptr(), presence.data_ptr(), count, dt, f,
                                      out.ctypes.data, out.size, offs.ctypes.data, C.byref(total)))
        return [out[int(offs[i]):int(offs[i + 1])].tobytes() for i in range(count)]

    def format_curve(self, thresholds, chi, fmt: str = "csv") -> bytes:
        """write_curve (fmt "csv" / "json", curve.hpp:87-121) or write_vcec
        ("vcec": values + changes, curve.hpp:154-169) bytes of ONE curve,
        formatted on the GPU -- f32 thresholds as std::to_chars' shortest
        round-trip text.  numpy arrays or CUDA tensors."""
        mode = {"csv": 0, "json": 1, "vcec": 2}[fmt]
        dev = hasattr(thresholds, "data_ptr")
        if dev:
            import torch
            dt = {torch.uint8: np.uint8, torch.uint16: np.uint16, torch.float32: np.float32}[thresholds.dtype]
            tp, cp, n = thresholds.data_ptr(), chi.data_ptr(), thresholds.numel()
        else:
            thresholds = np.ascontiguousarray(thresholds)
            chi = np.ascontiguousarray(chi, dtype=np.int64)
            dt, tp, cp, n = thresholds.dtype, thresholds.ctypes.data, chi.ctypes.data, thresholds.size
        total = _u64()
        rc = lib().ecc_format_curve(self._p, _DT[np.dtype(dt)], tp, cp, n, 1 if dev else 0, mode,
                                    None, 0, C.byref(total))
        if rc != 0 and total.value == 0:
            _check(rc)
        out = np.empty(max(1, total.value), np.uint8)
        _check(lib().ecc_format_curve(self._p, _DT[np.dtype(dt)], tp, cp, n, 1 if dev else 0, mode,
                                      out.ctypes.data, out.size, C.byref(total)))
        return out[:total.value].tobytes()

    def batch_zero_crossings(self, chi, presence, dtype=np.uint16, out=None, stream: int = 0):
        """zero_crossings (curve.hpp:36-50) of every image of a device batch:
        a (count, nbins/32) int32 bitmap tensor (bit t = occurring bin t is
        a zero crossing)."""
        import torch
        dt = _DT[np.dtype(dtype)]
        if out is None:
            out = torch.empty_like(presence)
        _check(lib().ecc_batch_zero_crossings(self._p, chi.data_ptr(), presence.data_ptr(),
                                              chi.shape[0], dt, out.data_ptr(), self._s(stream)))
        return out

    def fill_synthetic(self, tensor, seed: int = 1, base: int = 0, stream: int = 0):
        import torch
        dt = {torch.uint8: ECC_U8, torch.uint16: ECC_U16, torch.float32: ECC_F32}[tensor.dtype]
        _check(lib().ecc_fill_synthetic(self._p, tensor.data_ptr(), dt, tensor.numel(), seed, base,
                                        self._s(stream)))
        if not stream:  # a setup utility: done when it returns, visible to every stream
            torch.cuda.current_stream(self.device).synchronize()


_default_ctx = {}


@atexit.register
def _close_all():
    # destroy contexts before the CUDA runtime tears down at interpreter exit
    for c in list(_live):
        c.close()
    _default_ctx.clear()


def context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


def process_image(image, plan: ChunkPlan = None, options: EngineOptions = None,
                  report: EngineReport = None, binmap=None) -> GlobalVcec:
    """process_image (streaming.hpp:181-338).  A host array with a plan is
    streamed chunk by chunk through a MemorySource (the reference's Image
    overload); a device tensor or a host array without a plan runs as one
    resident volume."""
    options = options or EngineOptions()
    ctx = context(options.device)
    if isinstance(image, ChunkSource):
        if plan is None:
            plan = _even_plan(image.dims().w0, 1)
        return ctx.process_source(image, plan, options, report, binmap)
    if plan is not None and not _is_torch_cuda(image):
        arr = image if isinstance(image, np.ndarray) else np.asarray(image)
        sorted_f32 = arr.dtype == np.float32 and (binmap is None or
                                                  _binmap(ECC_F32, binmap).kind == ECC_BIN_SORTED)
        if not sorted_f32 and options.ingest_delay_ms <= 0:
            # the whole image is already in host memory: chunks are DMA-copied
            # straight from it (ecc_process_host), no read_rows round trip
            return ctx.process_host(arr, plan, report, binmap)
        return ctx.process_source(MemorySource(image), plan, options, report, binmap)
    return ctx.vcec(image, binmap)


class Exchange:
    """Fused multi-GPU rank exchange (ecc_xchg_*): create on every rank,
    all-gather `handle` (64 bytes), `open(handles)`, then
    Context.curve_sharded(...) runs K1+K2 over the rank's slab and the
    histogram exchange over peer memory + K3 in ONE launch."""

    def __init__(self, ctx: "Context", rank: int, world: int):
        self.ctx = ctx
        self._p = C.c_void_p()
        h = C.create_string_buffer(64)
        _check(lib().ecc_xchg_create(ctx._p, rank, world, C.byref(self._p), h))
        self.handle = h.raw
        self.world = world

    def open(self, handles):
        buf = b"".join(handles)
        assert len(buf) == 64 * self.world
        _check(lib().ecc_xchg_open(self._p, buf))

    def status(self):
        _check(lib().ecc_xchg_status(self._p))

    def close(self):
        if self._p:
            lib().ecc_xchg_destroy(self._p)
            self._p = C.c_void_p()


def _dims_of(shape) -> _Dims:
    d = Dims.of(shape)
    return _Dims(d.w0, d.w1, d.w2)


def bench_run(dims: Dims, iterations: int, seed: int = 1, sigma: float = 2.0, width: int = 13,
              device: int = 0) -> BenchReport:
    return context(device).bench_run(dims, iterations, seed, sigma, width)


def batch2d(images, **kw):
    return context().batch2d(images, **kw)


def curve_batch_to_points(chi_row: np.ndarray, presence_row: np.ndarray):
    """(thresholds, chi) of one batched image: the occurring bins only."""
    bits = np.unpackbits(presence_row.view(np.uint8), bitorder="little").astype(bool)
    t = np.nonzero(bits)[0]
    return t, chi_row[t].astype(np.int64)

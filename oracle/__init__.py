"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the ECC hot path.

Two checkers live here, both loaded through ctypes:

* ``liboracle.so`` -- ``ecc_oracle.c``, a plain-C restatement of the
  reference algorithm (each function cites the reference file:line it
  follows).
* ``_ref/libecc_ref.so`` -- the UNMODIFIED reference engine
  (``/root/reference/proj/include``) compiled in place by ``oracle/Makefile``
  (``make -C oracle ref``).  Used to pin the restatement, to generate the
  golden fixtures under ``tests/golden/`` and as the bench's reference arm.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline /
``--impl reference``) may import this module.  The product package
``paper_2203_09087_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

_u64 = C.c_uint64
_i64 = C.c_int64
_vp = C.c_void_p


def build(ref: bool = True) -> None:
    """Compile the C restatement (and the reference, when its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    if ref and os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        L.ecc_oracle_counter_hash.restype = _u64
        L.ecc_oracle_counter_hash.argtypes = [_u64, _u64]
        for n in ("ecc_oracle_fill_u8", "ecc_oracle_fill_u16", "ecc_oracle_fill_f32q"):
            getattr(L, n).argtypes = [_vp, _u64, _u64, _u64]
            getattr(L, n).restype = None
        for n in ("ecc_oracle_changes_u8", "ecc_oracle_changes_u16_as_f32",
                  "ecc_oracle_changes_f32"):
            getattr(L, n).argtypes = [_vp, _u64, _u64, _u64, _vp]
            getattr(L, n).restype = C.c_int
        for n in ("ecc_oracle_vcec_u8", "ecc_oracle_vcec_u16"):
            getattr(L, n).argtypes = [_vp, _u64, _u64, _u64, _vp, _vp]
            getattr(L, n).restype = C.c_int
        L.ecc_oracle_vcec_f32.argtypes = [_vp, _u64, _u64, _u64, _vp, _vp]
        L.ecc_oracle_vcec_f32.restype = _i64
        L.ecc_oracle_float_order_key.argtypes = [C.c_float]
        L.ecc_oracle_float_order_key.restype = C.c_uint32
        L.ecc_oracle_float_from_order_key.argtypes = [C.c_uint32]
        L.ecc_oracle_float_from_order_key.restype = C.c_float
        L.ecc_oracle_uniform_noise.argtypes = [_vp, _u64, _u64]
        L.ecc_oracle_uniform_noise.restype = None
        L.ecc_oracle_gaussian_smooth.argtypes = [_vp, _vp, _u64, _u64, _u64, C.c_double, C.c_int]
        L.ecc_oracle_gaussian_smooth.restype = C.c_int
        _LIB = L
    return _LIB


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libecc_ref.so"))


def ref():
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "libecc_ref.so")
        if not os.path.exists(path):
            raise FileNotFoundError("reference engine not built: make -C oracle ref")
        R = C.CDLL(path)
        R.ref_last_error.restype = C.c_char_p
        R.ref_hardware_concurrency.restype = C.c_uint
        R.ref_counter_hash.restype = _u64
        R.ref_counter_hash.argtypes = [_u64, _u64]
        for n in ("ref_vcec_u8", "ref_vcec_f32"):
            getattr(R, n).argtypes = [_vp, _u64, _u64, _u64, _u64, C.c_uint, _vp, _vp, _vp]
            getattr(R, n).restype = _i64
        for n in ("ref_naive_u8", "ref_naive_f32"):
            getattr(R, n).argtypes = [_vp, _u64, _u64, _u64, _vp, _vp]
            getattr(R, n).restype = _i64
        for n in ("ref_curve_csv_u8", "ref_curve_csv_f32"):
            getattr(R, n).argtypes = [_vp, _vp, _u64, _vp, _u64]
            getattr(R, n).restype = _i64
        R.ref_uniform_noise.argtypes = [_u64, _u64, _u64, _u64, _vp]
        R.ref_uniform_noise.restype = None
        R.ref_gaussian_smooth.argtypes = [_vp, _u64, _u64, _u64, C.c_double, C.c_int, _vp]
        R.ref_gaussian_smooth.restype = C.c_int
        R.ref_bench_run.argtypes = [_u64, _u64, _u64, _u64, _u64, C.c_double, C.c_int, _vp]
        R.ref_bench_run.restype = C.c_int
        _REF = R
    return _REF


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_vp)


# ---------------------------------------------------------------- inputs
def synth(kind: str, dims, seed: int = 1, base: int = 0) -> np.ndarray:
    """SURVEY.md 8(d) synthetic inputs (counter_hash, datagen.hpp:18-27)."""
    n = int(np.prod(dims))
    if kind == "u8":
        a = np.empty(n, np.uint8)
        lib().ecc_oracle_fill_u8(_p(a), n, seed, base)
    elif kind == "u16":
        a = np.empty(n, np.uint16)
        lib().ecc_oracle_fill_u16(_p(a), n, seed, base)
    elif kind == "f32q":
        a = np.empty(n, np.float32)
        lib().ecc_oracle_fill_f32q(_p(a), n, seed, base)
    else:
        raise ValueError(kind)
    return a.reshape(dims)


def _dims3(img: np.ndarray):
    if img.ndim == 2:
        return img.shape[0], img.shape[1], 1
    return img.shape


# ---------------------------------------------------------------- C restatement
def changes(img: np.ndarray) -> np.ndarray:
    """Per-voxel Euler changes (int8), row-major -- compute_changes."""
    img = np.ascontiguousarray(img)
    w0, w1, w2 = _dims3(img)
    out = np.empty(img.size, np.int8)
    fn = {np.dtype(np.uint8): "ecc_oracle_changes_u8",
          np.dtype(np.uint16): "ecc_oracle_changes_u16_as_f32",
          np.dtype(np.float32): "ecc_oracle_changes_f32"}[img.dtype]
    rc = getattr(lib(), fn)(_p(img), w0, w1, w2, _p(out))
    assert rc == 0
    return out.reshape(img.shape)


def vcec(img: np.ndarray):
    """(values, changes) of the global VCEC: ascending occurring values."""
    img = np.ascontiguousarray(img)
    w0, w1, w2 = _dims3(img)
    if img.dtype in (np.uint8, np.uint16):
        nb = 256 if img.dtype == np.uint8 else 65536
        hist = np.empty(nb, np.int64)
        cnt = np.empty(nb, np.int64)
        fn = lib().ecc_oracle_vcec_u8 if nb == 256 else lib().ecc_oracle_vcec_u16
        assert fn(_p(img), w0, w1, w2, _p(hist), _p(cnt)) == 0
        occ = np.nonzero(cnt)[0]
        return occ.astype(img.dtype), hist[occ]
    if img.dtype == np.float32:
        vals = np.empty(img.size, np.float32)
        ch = np.empty(img.size, np.int64)
        m = lib().ecc_oracle_vcec_f32(_p(img), w0, w1, w2, _p(vals), _p(ch))
        if m == -2:
            raise ValueError("NaN input")
        assert m > 0
        return vals[:m].copy(), ch[:m].copy()
    raise TypeError(img.dtype)


def curve(img: np.ndarray):
    """(thresholds, chi): vcec_to_ecc over vcec()."""
    v, c = vcec(img)
    return v, np.cumsum(c, dtype=np.int64)


def hist_dense(img: np.ndarray):
    """Dense (change-sum, count) per bin for integer images."""
    img = np.ascontiguousarray(img)
    w0, w1, w2 = _dims3(img)
    nb = 256 if img.dtype == np.uint8 else 65536
    hist = np.empty(nb, np.int64)
    cnt = np.empty(nb, np.int64)
    fn = lib().ecc_oracle_vcec_u8 if nb == 256 else lib().ecc_oracle_vcec_u16
    assert fn(_p(img), w0, w1, w2, _p(hist), _p(cnt)) == 0
    return hist, cnt


# ---------------------------------------------------------------- reference engine
def uniform_noise(shape, seed: int) -> np.ndarray:
    """uniform_noise (datagen.hpp:57-62) restated in C."""
    out = np.empty(shape, np.float32)
    lib().ecc_oracle_uniform_noise(_p(out), out.size, seed)
    return out


def gaussian_smooth(img: np.ndarray, sigma: float, width: int) -> np.ndarray:
    """gaussian_smooth (datagen.hpp:108-122) restated in C."""
    img = np.ascontiguousarray(img, dtype=np.float32)
    w0, w1, w2 = _dims3(img)
    out = np.empty_like(img)
    if lib().ecc_oracle_gaussian_smooth(_p(img), _p(out), w0, w1, w2, sigma, width) != 0:
        raise ValueError("Gaussian kernel width must be odd and >= 1")
    return out


def ref_uniform_noise(shape, seed: int) -> np.ndarray:
    w0, w1, w2 = (tuple(shape) + (1,))[:3] if len(shape) == 2 else tuple(shape)
    out = np.empty(shape, np.float32)
    ref().ref_uniform_noise(w0, w1, w2, seed, _p(out))
    return out


def ref_gaussian_smooth(img: np.ndarray, sigma: float, width: int) -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.float32)
    w0, w1, w2 = _dims3(img)
    out = np.empty_like(img)
    R = ref()
    if R.ref_gaussian_smooth(_p(img), w0, w1, w2, sigma, width, _p(out)) != 0:
        raise ValueError(R.ref_last_error().decode())
    return out


def ref_bench_run(shape, iterations: int, seed: int = 1, sigma: float = 2.0, width: int = 13):
    """bench_run (pipeline.hpp:236-291) through the compiled reference:
    dict of its BenchReport timings."""
    w0, w1, w2 = tuple(shape) if len(shape) == 3 else (shape[0], shape[1], 1)
    r = np.zeros(6, np.float64)
    R = ref()
    if R.ref_bench_run(w0, w1, w2, iterations, seed, sigma, width, _p(r)) != 0:
        raise ValueError(R.ref_last_error().decode())
    keys = ("generate_s", "total_s", "per_iteration_s", "ecc_avg_s", "smooth_avg_s", "ecc_gvox_per_s")
    return dict(zip(keys, map(float, r)))


def ref_vcec(img: np.ndarray, chunks: int = 1, workers: int = 1, phases=None):
    """process_image through the compiled reference (u8 and f32 paths).

    u16 images go through the reference's f32 path (exact), as SURVEY.md 0
    prescribes; the returned values are then cast back to uint16."""
    img = np.ascontiguousarray(img)
    w0, w1, w2 = _dims3(img)
    R = ref()
    ph = np.zeros(4, np.float64)
    back = None
    if img.dtype == np.uint16:
        back = np.uint16
        img = img.astype(np.float32)
    n = img.size
    if img.dtype == np.uint8:
        vals = np.empty(256, np.uint8)
        ch = np.empty(256, np.int64)
        m = R.ref_vcec_u8(_p(img), w0, w1, w2, chunks, workers, _p(vals), _p(ch), _p(ph))
    elif img.dtype == np.float32:
        cap = min(n, 1 << 32)
        vals = np.empty(cap, np.float32)
        ch = np.empty(cap, np.int64)
        m = R.ref_vcec_f32(_p(img), w0, w1, w2, chunks, workers, _p(vals), _p(ch), _p(ph))
    else:
        raise TypeError(img.dtype)
    if m < 0:
        raise RuntimeError(R.ref_last_error().decode())
    if phases is not None:
        phases[:] = ph
    v = vals[:m].copy()
    if back is not None:
        v = v.astype(back)
    return v, ch[:m].copy()


def ref_curve(img: np.ndarray, chunks: int = 1, workers: int = 1):
    v, c = ref_vcec(img, chunks, workers)
    return v, np.cumsum(c, dtype=np.int64)


def ref_naive(img: np.ndarray):
    """naive_ecc (oracle.hpp:80-107): brute-force cell counting."""
    img = np.ascontiguousarray(img)
    w0, w1, w2 = _dims3(img)
    R = ref()
    if img.dtype == np.uint8:
        t = np.empty(256, np.uint8)
        fn = R.ref_naive_u8
    else:
        img = img.astype(np.float32)
        t = np.empty(img.size, np.float32)
        fn = R.ref_naive_f32
    chi = np.empty(t.size, np.int64)
    m = fn(_p(img), w0, w1, w2, _p(t), _p(chi))
    if m < 0:
        raise RuntimeError(R.ref_last_error().decode())
    return t[:m].copy(), chi[:m].copy()


def ref_csv(thresholds: np.ndarray, chi: np.ndarray) -> bytes:
    """write_curve CSV bytes exactly as the reference formats them."""
    R = ref()
    t = np.ascontiguousarray(thresholds)
    chi = np.ascontiguousarray(chi, dtype=np.int64)
    if t.dtype == np.uint8:
        fn = R.ref_curve_csv_u8
    else:
        t = t.astype(np.float32)
        fn = R.ref_curve_csv_f32
    cap = 64 + 48 * len(t)
    buf = C.create_string_buffer(cap)
    n = fn(_p(t), _p(chi), len(t), buf, cap)
    assert n >= 0
    return buf.raw[:n]


def curve_digest(thresholds: np.ndarray, chi: np.ndarray) -> str:
    """Format-independent SHA-256 of a curve: thresholds as float64 LE
    followed by chi as int64 LE.  Used for golden fixtures on the GPU box,
    where the reference formatter is not available."""
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(thresholds, dtype="<f8").tobytes())
    h.update(np.ascontiguousarray(chi, dtype="<i8").tobytes())
    return h.hexdigest()

"""Python mirror of the reference's HE Mul entry points over the C-ABI.

The reference API is C++ (namespace ``hemul``, /root/reference/proj/core):
``make_params`` (params.cpp:64-74), ``Scheme::warm_level`` / ``he_mul`` /
``rescale`` (heaan.hpp:74-100, heaan.cpp:119-410) and the lower-level
``ntt_forward`` / ``crt_forward`` / ``rns_pointwise_mul`` / ``icrt_reordered``
(ntt.hpp:34-39, rns.hpp:62-85). This module binds ``libhemul_gpu.so``
(include/hemul_gpu.h) with ctypes and keeps the reference's names, argument
meaning and error kinds:

* modulus mismatch      -> ``ValueError("ciphertext modulus mismatch")``
  (std::invalid_argument, heaan.cpp:341-342)
* depth exhausted       -> ``RuntimeError("multiplicative depth exhausted")``
  (std::runtime_error, heaan.cpp:344-345)

Arrays are numpy ``uint64`` (host) or torch ``uint64`` CUDA tensors (device;
the call then stays on the device). Polynomials use the reference BigPoly
layout (n, limbs) little-endian 64-bit limbs; a leading batch axis is allowed.

There is no CPU fallback: importing works anywhere, but every computing call
needs the CUDA library and a GPU and raises ``HemulGpuError`` otherwise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from pathlib import Path
from typing import Any

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libhemul_gpu.so"

HEMUL_OK = 0
HEMUL_E_ARG = 1
HEMUL_E_MODULUS_MISMATCH = 2
HEMUL_E_DEPTH = 3
HEMUL_E_CUDA = 4
HEMUL_E_OOM = 5
HEMUL_E_NO_EVK = 6
HEMUL_E_IO = 7

STAGES = ("crt", "ntt", "intt", "icrt", "extra")  # counters.hpp:13
KERNEL_CLASSES = ("crt", "ntt_a", "ntt_b", "intt_b", "intt_a", "tensor", "evk", "icrt",
                  "finish", "mid_r1", "mid_r2", "epilogue", "h2d",
                  "d2h")  # HEMUL_KCLASS_* in include/hemul_gpu.h


class HemulGpuError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[status {status}] {message}")
        self.status = status


_lib: ctypes.CDLL | None = None

_u64p = ctypes.c_void_p
_SIGS = {
    "hemul_gpu_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_void_p)]),
    "hemul_gpu_destroy": (None, [ctypes.c_void_p]),
    "hemul_gpu_last_error": (ctypes.c_char_p, [ctypes.c_void_p]),
    "hemul_gpu_params": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]),
    "hemul_gpu_set_level": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "hemul_gpu_set_evk": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u64p, _u64p,
                                         ctypes.c_uint64]),
    "hemul_gpu_he_mul": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_size_t, _u64p, _u64p, _u64p, _u64p, _u64p,
                                        _u64p, ctypes.c_uint64, _u64p, _u64p]),
    "hemul_gpu_rescale": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, _u64p,
                                         _u64p, _u64p, _u64p]),
    "hemul_gpu_enable_stage_timing": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "hemul_gpu_stage_ms": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]),
    "hemul_gpu_level_twiddles32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "hemul_gpu_ntt32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]),
    "hemul_gpu_level_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_int), _u64p, ctypes.c_int]),
    "hemul_gpu_ntt": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _u64p,
                                     ctypes.c_size_t, ctypes.c_int]),
    "hemul_gpu_crt": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_size_t, _u64p, _u64p]),
    "hemul_gpu_pointwise": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_size_t, _u64p, _u64p, _u64p]),
    "hemul_gpu_icrt": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_size_t, _u64p, _u64p]),
    "hemul_gpu_launch_count": (ctypes.c_uint64, [ctypes.c_void_p]),
    "hemul_gpu_synchronize": (ctypes.c_int, [ctypes.c_void_p]),
    "hemul_ciphertext_digest": (ctypes.c_uint64, [ctypes.c_int, ctypes.c_size_t, _u64p, _u64p]),
    "hemul_gpu_set_stream": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "hemul_gpu_kernel_stats": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                              ctypes.POINTER(ctypes.c_uint64)]),
    "hemul_gpu_reset_stats": (ctypes.c_int, [ctypes.c_void_p]),
    "hemul_gpu_imad_peak": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]),
    "hemul_gpu_tc_peak": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]),
    "hemul_gpu_set_option": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
    "hemul_gpu_engine_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_int)]),
    "hemul_gpu_he_mul_trace": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t,
                                              _u64p, _u64p, _u64p, _u64p, _u64p, _u64p,
                                              ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p,
                                              ctypes.c_size_t,
                                              ctypes.POINTER(ctypes.c_size_t)]),
}
_SIGS.update({
    "hemul_gpu_ct_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, _u64p,
                                           _u64p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "hemul_gpu_ct_destroy": (None, [ctypes.c_void_p, ctypes.c_void_p]),
    "hemul_gpu_ct_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int),
                                         ctypes.POINTER(ctypes.c_size_t)]),
    "hemul_gpu_ct_device_ptrs": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p),
                                                ctypes.POINTER(ctypes.c_void_p)]),
    "hemul_gpu_ct_download": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _u64p, _u64p]),
    "hemul_gpu_ct_he_mul": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           _u64p, _u64p, ctypes.c_uint64,
                                           ctypes.POINTER(ctypes.c_void_p)]),
    "hemul_gpu_ct_rescale": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.POINTER(ctypes.c_void_p)]),
    "hemul_gpu_ct_mod_down": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_void_p)]),
})
_SIGS.update({
    "hemul_gpu_ct_load": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p,
                                         ctypes.POINTER(ctypes.c_void_p),
                                         ctypes.POINTER(ctypes.c_int)]),
    "hemul_gpu_ct_save": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                         ctypes.c_char_p]),
    "hemul_gpu_mul_by_ternary": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t,
                                                _u64p, ctypes.c_void_p, _u64p]),
})
HEMUL_OPT_LEVEL_CACHE = 4
ENGINE_INFO = ("word", "np1", "np2", "split_h", "crt1_tc", "crt2_tc", "big_tc", "fused_mid",
               "blk_mont", "t_pass_a")  # HEMUL_INFO_* in include/hemul_gpu.h
TRACE_POINTS = {"crt1": 1, "prod1": 2, "d2": 3, "crt2": 4, "prod2": 5}  # HEMUL_TRACE_*
HEMUL_OPT_FORCE_EXACT = 1
HEMUL_OPT_BASIS = 2
HEMUL_OPT_TENSOR_CORES = 3
HEMUL_OPT_TRANSPOSED = 5


def load_library(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load libhemul_gpu.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise HemulGpuError(HEMUL_E_CUDA, f"{p} missing: run `python -m paper_2003_04510_b200.build`")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


class DeviceCiphertext:
    """A batch of ciphertexts resident in device memory (hemul_gpu_ct): the
    operands of a device-resident HE Mul chain. Operations on it queue work
    on the context stream; ``download`` returns host arrays."""

    def __init__(self, ctx: "Context", handle: ctypes.c_void_p):
        self._ctx = ctx
        self._h = handle
        q = ctypes.c_int()
        b = ctypes.c_size_t()
        ctx._check(ctx._lib.hemul_gpu_ct_info(handle, ctypes.byref(q), ctypes.byref(b)))
        self.log_q = q.value
        self.batch = b.value

    @property
    def shape(self) -> tuple[int, ...]:
        n, L = self._ctx.n, limbs(self.log_q)
        return (self.batch, n, L) if self.batch > 1 else (n, L)

    def download(self, out: tuple[Any, Any] | None = None) -> tuple[Any, Any]:
        """(ax, bx) to host arrays (or into `out`: pinned host buffers make the
        copy run at full PCIe speed; device tensors work too)."""
        if out is None:
            out = (np.empty(self.shape, np.uint64), np.empty(self.shape, np.uint64))
        n_words = self.batch * self._ctx.n * limbs(self.log_q)
        if _size(out[0]) != n_words or _size(out[1]) != n_words:
            raise ValueError("download buffers do not match the ciphertext batch")
        self._ctx._check(self._ctx._lib.hemul_gpu_ct_download(self._ctx._h, self._h,
                                                              _ptr(out[0]), _ptr(out[1])))
        return out

    def device_ptrs(self) -> tuple[int, int]:
        a, b = ctypes.c_void_p(), ctypes.c_void_p()
        self._ctx._check(self._ctx._lib.hemul_gpu_ct_device_ptrs(self._h, ctypes.byref(a),
                                                                 ctypes.byref(b)))
        return a.value, b.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            ctx = self._ctx
            ctx._lib.hemul_gpu_ct_destroy(ctx._h if ctx._h else None, self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


@dataclass(frozen=True)
class Params:
    """make_params(log_p, depth, w64, log_n_override) (params.cpp:64-74)."""
    log_p: int
    depth: int
    log_n_override: int = 0

    @property
    def log_q_max(self) -> int:
        return self.log_p * self.depth

    @property
    def log_n(self) -> int:
        if self.log_n_override:
            return self.log_n_override
        q = self.log_q_max
        for bound, ln in ((300, 14), (600, 15), (1200, 16), (2400, 17)):
            if q <= bound:
                return ln
        raise ValueError("modulus too large for security table")

    @property
    def n(self) -> int:
        return 1 << self.log_n


def make_params(log_p: int, depth: int, log_n_override: int = 0) -> Params:
    return Params(log_p, depth, log_n_override)


def limbs(bits: int) -> int:
    return (bits + 63) // 64


def _ptr(a: Any, dtype: Any = np.uint64) -> int:
    """Raw address of a numpy array or torch tensor (contiguous, uint64 or
    the given numpy dtype)."""
    if isinstance(a, np.ndarray):
        if a.dtype != dtype or not a.flags["C_CONTIGUOUS"]:
            raise ValueError(f"expected a C-contiguous {np.dtype(dtype).name} numpy array")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("expected a contiguous tensor")
        return a.data_ptr()
    raise TypeError(f"unsupported buffer type {type(a)!r}")


def _like(a: Any, shape: tuple[int, ...]):
    if isinstance(a, np.ndarray):
        return np.empty(shape, dtype=np.uint64)
    import torch

    return torch.empty(shape, dtype=torch.uint64, device=a.device)


_CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy (driver_types.h)


def _size(a: Any) -> int:
    return int(a.size) if isinstance(a, np.ndarray) else int(a.numel())


class Context:
    """One device context = one reference ``Scheme`` (heaan.hpp:72-115) for
    the GPU path: parameters, a 2-entry level LRU, cached evk forms."""

    def __init__(self, params: Params, device: int = 0):
        self._lib = load_library()
        self.params = params
        h = ctypes.c_void_p()
        st = self._lib.hemul_gpu_create(device, params.log_p, params.depth,
                                        params.log_n_override, ctypes.byref(h))
        if st != HEMUL_OK:
            raise HemulGpuError(st, "hemul_gpu_create failed (no usable CUDA device?)")
        self._h = h
        # evk identity (see _evk_identity); automatic ids live above 2^62 so
        # they never meet explicit caller ids
        self._evk_last: tuple[Any, Any, int] | None = None
        self._evk_seq = 1 << 62
        # stream ordering with torch: until set_stream() names a stream, calls
        # that receive torch CUDA tensors run on torch's current stream (so
        # the producer of the inputs and the consumer of the outputs are
        # ordered with the library's kernels without a host sync)
        self._stream_explicit = False
        self._cur_stream: int | None = None

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.hemul_gpu_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- plumbing --------------------------------------------------------
    def _follow_torch(self, *bufs: Any) -> None:
        if self._stream_explicit:
            return
        for b in bufs:
            if b is not None and getattr(b, "is_cuda", False):
                import torch

                # torch's default stream reports handle 0, which the C side
                # reads as "the context's own stream": pass cudaStreamLegacy
                s = torch.cuda.current_stream(b.device).cuda_stream or _CUDA_STREAM_LEGACY
                if s != self._cur_stream:
                    self._check(self._lib.hemul_gpu_set_stream(self._h, s))
                    self._cur_stream = s
                return

    def _check(self, st: int) -> None:
        if st == HEMUL_OK:
            return
        msg = self._lib.hemul_gpu_last_error(self._h).decode()
        if st == HEMUL_E_MODULUS_MISMATCH:
            raise ValueError(msg)
        if st == HEMUL_E_DEPTH:
            raise RuntimeError(msg)
        raise HemulGpuError(st, msg)

    @property
    def n(self) -> int:
        return self.params.n

    # -- Scheme-level API ------------------------------------------------
    def _evk_identity(self, evk: tuple[Any, Any] | None, evk_id: int | None) -> int:
        """The id the C side keys its cached evk forms by. The reference keys
        them by the EvalKey's address (heaan.cpp:152); here by the identity of
        the two arrays: the same objects as last time keep their id (the
        context holds them, so the identity cannot be recycled), anything else
        gets a fresh one. An explicit evk_id overrides (0 = always rebuild)."""
        if evk is None:
            return 0
        if evk_id is not None:
            return int(evk_id)
        last = self._evk_last
        if last is not None and last[0] is evk[0] and last[1] is evk[1]:
            return last[2]
        self._evk_seq += 1
        self._evk_last = (evk[0], evk[1], self._evk_seq)
        return self._evk_seq

    def warm_level(self, log_q: int, evk: tuple[Any, Any] | None = None,
                   evk_id: int | None = None) -> None:
        """Scheme::warm_level (heaan.hpp:100): tables, and evk forms if given."""
        self._follow_torch(*(evk or ()))
        if evk is None:
            self._check(self._lib.hemul_gpu_set_level(self._h, log_q))
        else:
            ea, eb = evk
            self._check(self._lib.hemul_gpu_set_evk(self._h, log_q, _ptr(ea), _ptr(eb),
                                                    self._evk_identity(evk, evk_id)))

    def he_mul(self, c1: tuple[Any, Any], c2: tuple[Any, Any], log_q: int,
               c2_log_q: int | None = None, evk: tuple[Any, Any] | None = None,
               evk_id: int | None = None, out: tuple[Any, Any] | None = None):
        """Scheme::he_mul (heaan.cpp:339-410) on (ax, bx) pairs. Inputs have
        shape (n, limbs) or (batch, n, limbs); returns (ax, bx) at modulus
        log_q - log_p."""
        self._follow_torch(c1[0], c2[0], *(evk or ()), *(out or ()))
        c2_log_q = log_q if c2_log_q is None else c2_log_q
        p = self.params
        if log_q != c2_log_q:
            self._check(self._lib.hemul_gpu_he_mul(self._h, log_q, c2_log_q, 1, None, None, None,
                                                   None, None, None, 0, None, None))
        L, Lo = limbs(log_q), limbs(log_q - p.log_p)
        per = self.n * L
        total = _size(c1[0])
        if total % per:
            raise ValueError("ciphertext buffer is not a multiple of n x limbs")
        batch = total // per
        for a in (c1[1], c2[0], c2[1]):
            if _size(a) != total:
                raise ValueError("ciphertext components differ in size")
        shape = (batch, self.n, Lo) if batch > 1 or getattr(c1[0], "ndim", 2) == 3 else (self.n, Lo)
        if out is None:
            out = (_like(c1[0], shape), _like(c1[0], shape))
        ea = _ptr(evk[0]) if evk is not None else None
        eb = _ptr(evk[1]) if evk is not None else None
        self._check(self._lib.hemul_gpu_he_mul(
            self._h, log_q, c2_log_q, batch, _ptr(c1[0]), _ptr(c1[1]), _ptr(c2[0]), _ptr(c2[1]),
            ea, eb, self._evk_identity(evk, evk_id), _ptr(out[0]), _ptr(out[1])))
        return out

    def rescale(self, c: tuple[Any, Any], log_q: int):
        """Scheme::rescale (heaan.cpp:328-337)."""
        self._follow_torch(c[0])
        p = self.params
        L, Lo = limbs(log_q), limbs(log_q - p.log_p)
        batch = _size(c[0]) // (self.n * L)
        shape = (batch, self.n, Lo) if batch > 1 else (self.n, Lo)
        out = (_like(c[0], shape), _like(c[0], shape))
        self._check(self._lib.hemul_gpu_rescale(self._h, log_q, batch, _ptr(c[0]), _ptr(c[1]),
                                                _ptr(out[0]), _ptr(out[1])))
        return out

    # -- device-resident chains (hemul_gpu_ct_*) -----------------------------
    def upload(self, c: tuple[Any, Any], log_q: int, asynchronous: bool = False) -> DeviceCiphertext:
        """Ciphertext(s) (ax, bx) of shape (n, limbs) or (batch, n, limbs) into
        device memory. asynchronous=True queues the copy on the copy stream
        (HEMUL_CT_ASYNC): the sources must stay alive and unchanged until the
        next download / synchronize."""
        self._follow_torch(c[0])
        per = self.n * limbs(log_q)
        batch = _size(c[0]) // per
        if batch * per != _size(c[0]) or _size(c[1]) != _size(c[0]):
            raise ValueError("ciphertext buffers are not batch x n x limbs")
        h = ctypes.c_void_p()
        self._check(self._lib.hemul_gpu_ct_create(self._h, log_q, batch, _ptr(c[0]), _ptr(c[1]),
                                                  int(asynchronous), ctypes.byref(h)))
        return DeviceCiphertext(self, h)

    def he_mul_dev(self, c1: DeviceCiphertext, c2: DeviceCiphertext,
                   evk: tuple[Any, Any] | None = None,
                   evk_id: int | None = None) -> DeviceCiphertext:
        """Scheme::he_mul on device-resident operands; the result stays on the device."""
        self._follow_torch(*(evk or ()))
        h = ctypes.c_void_p()
        ea = _ptr(evk[0]) if evk is not None else None
        eb = _ptr(evk[1]) if evk is not None else None
        self._check(self._lib.hemul_gpu_ct_he_mul(self._h, c1._h, c2._h, ea, eb,
                                                  self._evk_identity(evk, evk_id), ctypes.byref(h)))
        return DeviceCiphertext(self, h)

    def rescale_dev(self, c: DeviceCiphertext) -> DeviceCiphertext:
        h = ctypes.c_void_p()
        self._check(self._lib.hemul_gpu_ct_rescale(self._h, c._h, ctypes.byref(h)))
        return DeviceCiphertext(self, h)

    def mod_down_dev(self, c: DeviceCiphertext, new_log_q: int) -> DeviceCiphertext:
        """poly_mod_down (poly.cpp:117-127) of both polynomials."""
        h = ctypes.c_void_p()
        self._check(self._lib.hemul_gpu_ct_mod_down(self._h, c._h, new_log_q, ctypes.byref(h)))
        return DeviceCiphertext(self, h)

    def load_dev(self, path: str) -> tuple[DeviceCiphertext, int]:
        """HEA1 ciphertext file (io.cpp:101-141) straight into HBM; returns
        (handle, n_slots)."""
        h = ctypes.c_void_p()
        slots = ctypes.c_int()
        self._check(self._lib.hemul_gpu_ct_load(self._h, str(path).encode(), ctypes.byref(h),
                                                ctypes.byref(slots)))
        return DeviceCiphertext(self, h), slots.value

    def save_dev(self, c: DeviceCiphertext, path: str, n_slots: int = 0) -> None:
        self._check(self._lib.hemul_gpu_ct_save(self._h, c._h, n_slots, str(path).encode()))

    def mul_by_ternary(self, a: np.ndarray, t: np.ndarray, log_q: int) -> np.ndarray:
        """Scheme::mul_by_ternary (heaan.cpp:234-256) on the GPU."""
        a = np.ascontiguousarray(a, dtype=np.uint64)
        t = np.ascontiguousarray(t, dtype=np.int32)
        out = np.empty_like(a)
        batch = a.size // (self.n * limbs(log_q))
        self._check(self._lib.hemul_gpu_mul_by_ternary(self._h, log_q, batch, a.ctypes.data,
                                                       t.ctypes.data, out.ctypes.data))
        return out

    def set_level_cache(self, capacity: int) -> None:
        """Level LRU capacity (default 2 like Scheme::level, heaan.cpp:119-150)."""
        self._check(self._lib.hemul_gpu_set_option(self._h, HEMUL_OPT_LEVEL_CACHE, capacity))

    def engine_info(self, log_q: int) -> dict[str, int]:
        """Basis and kernels he_mul uses at level log_q (hemul_gpu_engine_info)."""
        buf = (ctypes.c_int * len(ENGINE_INFO))()
        self._check(self._lib.hemul_gpu_engine_info(self._h, log_q, buf))
        return dict(zip(ENGINE_INFO, list(buf)))

    def he_mul_trace(self, c1: tuple[Any, Any], c2: tuple[Any, Any], log_q: int, point: str,
                     evk: tuple[Any, Any] | None = None, evk_id: int | None = None) -> np.ndarray:
        """Test hook: he_mul stopped at a stage checkpoint (crt1, prod1, d2,
        crt2, prod2; include/hemul_gpu.h HEMUL_TRACE_*); returns that stage's
        buffer (uint32 residues in the 30-bit basis, uint64 otherwise)."""
        self._follow_torch(c1[0], c2[0], *(evk or ()))
        info = self.engine_info(log_q)
        p = self.params
        per = self.n * limbs(log_q)
        batch = _size(c1[0]) // per
        w = 4 if info["word"] == 32 else 8
        rows = {"crt1": (8 if w == 4 else 4) * batch * info["np1"],
                "prod1": (6 if w == 4 else 3) * batch * info["np1"],
                "crt2": batch * info["np2"], "prod2": 2 * batch * info["np2"]}
        if point == "d2":
            out = np.zeros((batch, self.n, limbs(log_q)), np.uint64)
        else:
            out = np.zeros((rows[point], self.n), np.uint32 if w == 4 else np.uint64)
        ea = _ptr(evk[0]) if evk is not None else None
        eb = _ptr(evk[1]) if evk is not None else None
        wrote = ctypes.c_size_t()
        self._check(self._lib.hemul_gpu_he_mul_trace(
            self._h, log_q, batch, _ptr(c1[0]), _ptr(c1[1]), _ptr(c2[0]), _ptr(c2[1]), ea, eb,
            self._evk_identity(evk, evk_id), TRACE_POINTS[point], out.ctypes.data, out.nbytes,
            ctypes.byref(wrote)))
        assert wrote.value == out.nbytes, (wrote.value, out.nbytes)
        del p
        return out

    # -- stage API (ntt.hpp / rns.hpp) -------------------------------------
    def level_primes(self, log_q: int, region: int) -> np.ndarray:
        np_ = ctypes.c_int()
        self._check(self._lib.hemul_gpu_level_info(self._h, log_q, region, ctypes.byref(np_),
                                                   None, 0))
        buf = np.zeros(np_.value, dtype=np.uint64)
        self._check(self._lib.hemul_gpu_level_info(self._h, log_q, region, ctypes.byref(np_),
                                                   buf.ctypes.data, np_.value))
        return buf

    def level_twiddles32(self, log_q: int, region: int, j: int) -> tuple[np.ndarray, np.ndarray]:
        """(tw, itw) of prime j of the level's 30-bit basis: (n, 2) u32 (w, wq)."""
        tw = np.zeros((self.n, 2), np.uint32)
        itw = np.zeros((self.n, 2), np.uint32)
        self._check(self._lib.hemul_gpu_level_twiddles32(self._h, log_q, region, j,
                                                         tw.ctypes.data, itw.ctypes.data))
        return tw, itw

    def ntt32(self, data: Any, log_q: int, region: int, inverse: bool = False,
              nprimes: int = 0) -> None:
        """The 30-bit basis NTT of the he_mul path, in place over u32 rows
        (row r mod level_primes(log_q, -region)[r % nprimes]; 0 = all)."""
        self._follow_torch(data)
        rows = _size(data) // self.n
        self._check(self._lib.hemul_gpu_ntt32(self._h, log_q, region, nprimes,
                                              _ptr(data, np.uint32), rows, int(inverse)))

    def ntt(self, data: Any, log_q: int, region: int, inverse: bool = False) -> None:
        """In place over rows of n residues (row r uses prime r % np)."""
        self._follow_torch(data)
        rows = _size(data) // self.n
        self._check(self._lib.hemul_gpu_ntt(self._h, log_q, region, _ptr(data), rows, int(inverse)))

    def crt(self, poly: Any, log_q: int, region: int, in_bits: int):
        self._follow_torch(poly)
        batch = _size(poly) // (self.n * limbs(in_bits))
        np_ = len(self.level_primes(log_q, region))
        out = _like(poly, (batch, np_, self.n) if batch > 1 else (np_, self.n))
        self._check(self._lib.hemul_gpu_crt(self._h, log_q, region, in_bits, batch, _ptr(poly),
                                            _ptr(out)))
        return out

    def pointwise(self, a: Any, b: Any, log_q: int, region: int):
        self._follow_torch(a, b)
        np_ = len(self.level_primes(log_q, region))
        batch = _size(a) // (np_ * self.n)
        out = _like(a, tuple(a.shape))
        self._check(self._lib.hemul_gpu_pointwise(self._h, log_q, region, batch, _ptr(a), _ptr(b),
                                                  _ptr(out)))
        return out

    def icrt(self, rns: Any, log_q: int, region: int):
        self._follow_torch(rns)
        p = self.params
        np_ = len(self.level_primes(log_q, region))
        batch = _size(rns) // (np_ * self.n)
        tbits = log_q if region == 1 else log_q + p.log_q_max
        out = _like(rns, (batch, self.n, limbs(tbits)) if batch > 1 else (self.n, limbs(tbits)))
        self._check(self._lib.hemul_gpu_icrt(self._h, log_q, region, batch, _ptr(rns), _ptr(out)))
        return out

    # -- instrumentation ---------------------------------------------------
    def enable_stage_timing(self, on: bool = True) -> None:
        self._check(self._lib.hemul_gpu_enable_stage_timing(self._h, int(on)))

    def stage_ms(self) -> dict[str, float]:
        buf = (ctypes.c_double * 5)()
        self._check(self._lib.hemul_gpu_stage_ms(self._h, buf))
        return dict(zip(STAGES, list(buf)))

    def kernel_stats(self) -> dict[str, tuple[float, int]]:
        """Cumulative (ms, launches) per kernel class since reset_stats()."""
        k = len(KERNEL_CLASSES)
        ms = (ctypes.c_double * k)()
        n = (ctypes.c_uint64 * k)()
        self._check(self._lib.hemul_gpu_kernel_stats(self._h, ms, n))
        return {name: (ms[i], int(n[i])) for i, name in enumerate(KERNEL_CLASSES)}

    def reset_stats(self) -> None:
        self._check(self._lib.hemul_gpu_reset_stats(self._h))

    def set_force_exact(self, on: bool = True) -> None:
        """Route every he_mul output coefficient through the exact big-integer
        fix-up kernel (test knob for the rarely taken exact path)."""
        self._check(self._lib.hemul_gpu_set_option(self._h, HEMUL_OPT_FORCE_EXACT, int(on)))

    def set_basis(self, word: int) -> None:
        """RNS basis he_mul computes in: 32 (30-bit primes, default) or 64 (the
        reference's w64 primes). Bit-identical results; pass the evk to the
        next he_mul after switching."""
        self._check(self._lib.hemul_gpu_set_option(self._h, HEMUL_OPT_BASIS, int(word)))

    def set_tensor_cores(self, on: bool = True) -> None:
        """30-bit basis: run the big-integer base conversions as exact int8
        GEMMs on the tcgen05 tensor cores (default) or on the IMAD.WIDE
        integer pipe. Bit-identical results."""
        self._check(self._lib.hemul_gpu_set_option(self._h, HEMUL_OPT_TENSOR_CORES, int(on)))

    def set_transposed(self, on: bool = True) -> None:
        """Tensor-core engine, log N >= 15: column-major RNS rows around NTT
        pass A (HEMUL_OPT_TRANSPOSED). Bit-identical results."""
        self._check(self._lib.hemul_gpu_set_option(self._h, HEMUL_OPT_TRANSPOSED, int(on)))

    def mul_basis(self, log_q: int) -> tuple[int, int, int]:
        """(word, np1, np2) of the basis he_mul uses at level log_q."""
        p1 = self.level_primes(log_q, -1)
        p2 = self.level_primes(log_q, -2)
        word = 32 if int(p1.max()) < (1 << 30) else 64
        return word, len(p1), len(p2)

    def set_stream(self, stream: int | None) -> None:
        """Launch on this cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
        None: the context's own stream, and calls with torch CUDA tensors
        follow torch's current stream again."""
        self._check(self._lib.hemul_gpu_set_stream(self._h, stream))
        self._stream_explicit = stream is not None
        self._cur_stream = stream

    def imad_peak(self) -> float:
        """Measured IMAD.WIDE.U32 ops/s of this device."""
        v = ctypes.c_double()
        self._check(self._lib.hemul_gpu_imad_peak(self._h, ctypes.byref(v)))
        return v.value

    def tc_peak(self) -> float:
        """Measured dense int8 tensor-core ops/s (tcgen05.mma kind::i8) of this device."""
        v = ctypes.c_double()
        self._check(self._lib.hemul_gpu_tc_peak(self._h, ctypes.byref(v)))
        return v.value

    def launch_count(self) -> int:
        return int(self._lib.hemul_gpu_launch_count(self._h))

    def synchronize(self) -> None:
        self._check(self._lib.hemul_gpu_synchronize(self._h))


def ciphertext_digest(log_q: int, ax: np.ndarray, bx: np.ndarray) -> int:
    """FNV-1a 64 over log_q, ax words, bx words (bench.cpp:35-47)."""
    ax = np.ascontiguousarray(ax, dtype=np.uint64)
    bx = np.ascontiguousarray(bx, dtype=np.uint64)
    if ax.size != bx.size:
        raise ValueError("ax and bx differ in size")
    return int(load_library().hemul_ciphertext_digest(log_q, ax.size, ax.ctypes.data,
                                                      bx.ctypes.data))

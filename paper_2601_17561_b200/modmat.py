"""Python mirror of the reference's `irislab::modmat` API
(/root/reference/proj/include/irislab/modmat.hpp:11-93), executed by the
B200 engine through the C ABI. Same names, argument meaning, return values
and exception types; the arithmetic runs in libirl_b200.so's sm_100a kernels.

Types follow the reference: SmallMatrix is a row-major int32 matrix
(numpy array of shape (rows, cols)), BigMatrix holds Python ints in [0, Q).
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import capi


# --- errors (reference include/irislab/errors.hpp:9-53) ------------------------

class Error(RuntimeError):
    pass


class ShapeMismatch(Error):
    pass


class ModulusTooLarge(Error):
    pass


class AccumulationOverflowRisk(Error):
    pass


class ModulusBudget(Error):
    pass


class ZeroOverlap(Error):
    """errors.hpp:18-20: mask overlap is empty, score undefined."""


class ConfigError(Error):
    """errors.hpp:13-16: invalid pipeline / chain configuration."""


class DeviceError(Error):
    """CUDA / device failures (no reference counterpart)."""


_STATUS_EXC = {
    capi.IRL_ERR_SHAPE_MISMATCH: ShapeMismatch,
    capi.IRL_ERR_MODULUS_TOO_LARGE: ModulusTooLarge,
    capi.IRL_ERR_ACCUMULATION_OVERFLOW_RISK: AccumulationOverflowRisk,
    capi.IRL_ERR_NOT_COPRIME: Error,
    capi.IRL_ERR_MODULUS_BUDGET: ModulusBudget,
    capi.IRL_ERR_ZERO_OVERLAP: ZeroOverlap,
    capi.IRL_ERR_IO: Error,
    capi.IRL_ERR_CONFIG: ConfigError,
}


# --- context --------------------------------------------------------------------

class Context:
    """One device context (stream + workspace) of the engine."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        st = capi.lib().irl_ctx_create(device, C.byref(h))
        if st != capi.IRL_OK:
            raise DeviceError(f"irl_ctx_create(device={device}) failed: "
                              f"{capi.lib().irl_status_string(st).decode()} (needs an sm_100 GPU)")
        self.handle = h
        self.device = device

    def check(self, st: int):
        if st == capi.IRL_OK:
            return
        msg = capi.lib().irl_last_error(self.handle).decode()
        exc = _STATUS_EXC.get(st)
        if exc is None:
            raise DeviceError(f"{capi.lib().irl_status_string(st).decode()}: {msg}")
        raise exc(msg)

    @property
    def launches(self) -> int:
        return int(capi.lib().irl_kernel_launches(self.handle))

    @classmethod
    def borrowed(cls, handle, device: int) -> "Context":
        """A view of a context owned elsewhere (e.g. a rank of an irl_ccmm_group)."""
        self = cls.__new__(cls)
        self.handle, self.device, self._borrowed = handle, device, True
        return self

    def close(self):
        if self.handle and not getattr(self, "_borrowed", False):
            capi.lib().irl_ctx_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: Optional[Context] = None
_lock = threading.Lock()


def default_context() -> Context:
    global _default
    with _lock:
        if _default is None:
            _default = Context(0)
        return _default


# --- RNS basis (modmat.hpp:14-40, modmat.cpp:8-63) ---------------------------------

def primes_in_range(lo: int, hi: int) -> List[int]:
    out = []
    for n in range(max(lo, 2), hi + 1):
        if all(n % q for q in range(2, int(math.isqrt(n)) + 1)):
            out.append(n)
    return out


@dataclass
class Modulus:
    p: int = 0
    e: int = 1

    def value(self) -> int:
        return self.p * self.p if self.e == 2 else self.p


@dataclass
class RnsBasis:
    moduli: List[Modulus] = field(default_factory=list)
    Q: int = 1

    def digit_planes(self) -> int:
        return sum(m.e for m in self.moduli)

    def log2_Q(self) -> float:
        # exact: bit length plus log2 of the leading 53-bit mantissa
        shift = max(self.Q.bit_length() - 53, 0)
        return math.log2(self.Q >> shift) + shift

    def arrays(self):
        p = np.array([m.p for m in self.moduli], np.uint32)
        e = np.array([m.e for m in self.moduli], np.uint32)
        return p, e

    def width(self) -> int:
        """ceil(log256 Q): bytes per serialized entry (modmat.cpp:219)."""
        return max((self.Q.bit_length() + 7) // 8, 1)


def build_paper_basis() -> RnsBasis:
    b = RnsBasis()
    for p in primes_in_range(127, 253):
        b.moduli.append(Modulus(p, 2))
        b.Q *= p * p
    return b


def max_int8_rns_capacity() -> float:
    total = 0.0
    for p in primes_in_range(3, 253):
        e, pw = 0, 1
        while pw * p < 256:
            pw *= p
            e += 1
        total += e * math.log2(p)
    return total


def pure_rns_plane_count() -> int:
    return len(primes_in_range(3, 253))


# --- matrices --------------------------------------------------------------------

def SmallMatrix(rows: int, cols: int, a=None) -> np.ndarray:
    """Row-major int32 matrix (modmat.hpp:43-50)."""
    if a is None:
        return np.zeros((rows, cols), np.int32)
    return np.asarray(a, dtype=np.int32).reshape(rows, cols)


@dataclass
class DigitMatrices:
    p: int
    m0: np.ndarray
    m1: np.ndarray


class BigMatrix:
    """Row-major matrix of integers in [0, Q) (modmat.hpp:60-70)."""

    def __init__(self, rows: int, cols: int, a: Optional[List[int]] = None):
        self.rows, self.cols = rows, cols
        self.a = list(a) if a is not None else [0] * (rows * cols)

    @staticmethod
    def zeros(r: int, c: int) -> "BigMatrix":
        return BigMatrix(r, c)

    @staticmethod
    def identity(n: int) -> "BigMatrix":
        m = BigMatrix(n, n)
        for i in range(n):
            m.a[i * n + i] = 1
        return m

    def at(self, r: int, c: int) -> int:
        return self.a[r * self.cols + c]

    def reduce(self, Q: int):
        self.a = [x % Q for x in self.a]

    def to_le(self, width: int) -> np.ndarray:
        out = np.zeros((len(self.a), width), np.uint8)
        for i, v in enumerate(self.a):
            out[i] = np.frombuffer(int(v).to_bytes(width, "little"), np.uint8)
        return out

    @staticmethod
    def from_le(rows: int, cols: int, buf: np.ndarray, width: int) -> "BigMatrix":
        flat = np.ascontiguousarray(buf).reshape(-1, width)
        return BigMatrix(rows, cols, [int.from_bytes(bytes(r), "little") for r in flat])


# --- hot path ---------------------------------------------------------------------

def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.int32)


def digit_decompose(m, p: int, ctx: Optional[Context] = None) -> DigitMatrices:
    """modmat.cpp:86-106 on the GPU."""
    ctx = ctx or default_context()
    m = _i32(m)
    rows, cols = m.shape
    d0 = np.zeros_like(m)
    d1 = np.zeros_like(m)
    ctx.check(capi.lib().irl_digit_decompose(ctx.handle, capi.ptr(m, capi.i32p), rows, cols, p,
                                             capi.ptr(d0, capi.i32p), capi.ptr(d1, capi.i32p)))
    return DigitMatrices(p, d0, d1)


def digit_recompose(d: DigitMatrices, ctx: Optional[Context] = None) -> np.ndarray:
    """modmat.cpp:108-118 on the GPU."""
    ctx = ctx or default_context()
    m0, m1 = _i32(d.m0), _i32(d.m1)
    if m0.shape != m1.shape:
        raise ShapeMismatch("digit planes differ in shape")
    out = np.zeros_like(m0)
    ctx.check(capi.lib().irl_digit_recompose(ctx.handle, capi.ptr(m0, capi.i32p), capi.ptr(m1, capi.i32p),
                                             m0.shape[0], m0.shape[1], d.p, capi.ptr(out, capi.i32p)))
    return out


def small_gemm(a, b, ctx: Optional[Context] = None) -> np.ndarray:
    """modmat.cpp:120-141: int32 product with the same overflow precheck."""
    ctx = ctx or default_context()
    a, b = _i32(a), _i32(b)
    if a.shape[1] != b.shape[0]:
        raise ShapeMismatch("small_gemm: inner dimensions differ")
    c = np.zeros((a.shape[0], b.shape[1]), np.int32)
    ctx.check(capi.lib().irl_small_gemm(ctx.handle, capi.ptr(a, capi.i32p), capi.ptr(b, capi.i32p),
                                        capi.ptr(c, capi.i32p), a.shape[0], a.shape[1], b.shape[1]))
    return c


def gemm_mod_psq(a, b, p: int, ctx: Optional[Context] = None) -> np.ndarray:
    """modmat.cpp:143-160: A B mod p^2 via three fused int8 tensor-core GEMMs."""
    ctx = ctx or default_context()
    a, b = _i32(a), _i32(b)
    if a.shape[1] != b.shape[0]:
        # the reference reports this from small_gemm (modmat.cpp:121)
        if p >= 256:
            raise ModulusTooLarge("digit base must be < 2^8")
        raise ShapeMismatch("small_gemm: inner dimensions differ")
    c = np.zeros((a.shape[0], b.shape[1]), np.int32)
    ctx.check(capi.lib().irl_gemm_mod_psq(ctx.handle, capi.ptr(a, capi.i32p), capi.ptr(b, capi.i32p),
                                          capi.ptr(c, capi.i32p), a.shape[0], a.shape[1], b.shape[1], p))
    return c


def gemm_mod_Q(a: BigMatrix, b: BigMatrix, basis: RnsBasis, ctx: Optional[Context] = None) -> BigMatrix:
    """modmat.cpp:162-195: residues, per-modulus PPMMs, CRT — all on the GPU."""
    ctx = ctx or default_context()
    if a.cols != b.rows:
        raise ShapeMismatch("gemm_mod_Q: inner dimensions differ")
    w = basis.width()
    return BigMatrix.from_le(a.rows, b.cols, gemm_mod_Q_le(a.to_le(w), b.to_le(w), a.rows, a.cols, b.cols,
                                                           w, basis, ctx), w)


def gemm_mod_Q_le(a_le: np.ndarray, b_le: np.ndarray, m: int, k: int, n: int, width: int,
                  basis: RnsBasis, ctx: Optional[Context] = None) -> np.ndarray:
    """gemm_mod_Q on fixed-width little-endian entries (the file-format layout)."""
    ctx = ctx or default_context()
    p, e = basis.arrays()
    a_le = np.ascontiguousarray(a_le, np.uint8)
    b_le = np.ascontiguousarray(b_le, np.uint8)
    c = np.zeros((m * n, width), np.uint8)
    ctx.check(capi.lib().irl_gemm_mod_Q(ctx.handle, capi.ptr(a_le, capi.u8p), capi.ptr(b_le, capi.u8p),
                                        capi.ptr(c, capi.u8p), m, k, n, width, capi.ptr(p, capi.u32p),
                                        capi.ptr(e, capi.u32p), len(p)))
    return c


# --- serialization (modmat.cpp:216-249) ---------------------------------------------

def save_big_matrix(path: str, m: BigMatrix, Q: int):
    """Header `rows cols Q\\n`, then ceil(log256 Q)-byte little-endian entries."""
    width = max((Q.bit_length() + 7) // 8, 1)
    with open(path, "wb") as f:
        f.write(f"{m.rows} {m.cols} {Q}\n".encode())
        f.write(m.to_le(width).tobytes())


def load_big_matrix(path: str):
    """Returns (BigMatrix, Q)."""
    with open(path, "rb") as f:
        blob = f.read()
    nl = blob.index(b"\n")
    rows, cols, q = blob[:nl].split()
    rows, cols, Q = int(rows), int(cols), int(q)
    width = max((Q.bit_length() + 7) // 8, 1)
    body = blob[nl + 1:]
    if len(body) < rows * cols * width:
        raise Error(f"truncated matrix file {path}")
    buf = np.frombuffer(body[:rows * cols * width], np.uint8)
    return BigMatrix.from_le(rows, cols, buf, width), Q

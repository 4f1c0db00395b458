"""Host mirror of the reference's plaintext iris scoring (irislab::iris,
iris_core.hpp / iris_core.cpp, and the overlaps of pipeline::prepare,
pipeline.cpp:92-153) on the B200 engine (C ABI irl_iris_*, csrc/iris.cu).

Templates are numpy uint8 {0,1} arrays (code, mask) of length d, like the
reference's IrisTemplate. Every sum is computed by the tcgen05 kernel; this
module only packs bits (pack_bits, pipeline.cpp:70-76) and calls the ABI.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import capi
from .modmat import Context, ShapeMismatch, ZeroOverlap, default_context


@dataclass
class IrisTemplate:
    """iris_core.hpp: code and mask bits of the same length d."""
    code: np.ndarray
    mask: np.ndarray

    def size(self) -> int:
        return int(self.code.shape[0])

    def validate(self):
        # IrisTemplate::validate (iris_core.cpp:10-19)
        if self.code.shape != self.mask.shape or self.code.size == 0:
            raise ShapeMismatch("code and mask must have identical nonzero length")
        if (self.code > 1).any() or (self.mask > 1).any():
            raise ShapeMismatch("template entries must be bits")


@dataclass
class Interval:
    lo: float = 0.0
    hi: float = 0.0

    def contains(self, x: float) -> bool:
        return self.lo <= x <= self.hi


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """[n][d] {0,1} -> [n][ceil(d/64)] uint64, bit i of a row at word i/64,
    bit i%64 (pipeline.cpp:70-76)."""
    bits = np.ascontiguousarray(bits, np.uint8)
    n, d = bits.shape
    words = (d + 63) // 64
    padded = np.zeros((n, words * 64), np.uint8)
    padded[:, :d] = bits
    return np.packbits(padded.reshape(n, words, 8, 8)[:, :, ::-1, ::-1].reshape(n, words * 64),
                       axis=1, bitorder="big").view(">u8").astype(np.uint64).reshape(n, words)


def _stack(ts: Sequence[IrisTemplate]):
    d = ts[0].size() if ts else 0
    for t in ts:
        if t.size() != d:
            raise ShapeMismatch("template lengths differ")
    code = np.stack([t.code for t in ts]).astype(np.uint8) if ts else np.zeros((0, d), np.uint8)
    mask = np.stack([t.mask for t in ts]).astype(np.uint8) if ts else np.zeros((0, d), np.uint8)
    return pack_bits(code), pack_bits(mask), d


def _p(a):
    return capi.ptr(a) if a is not None and a.size else None


def inner_overlap(db: Sequence[IrisTemplate], eyes: Sequence[IrisTemplate], rho: int = 1,
                  ctx: Optional[Context] = None):
    """(inner, overlap), each int32 [len(eyes)*rho][len(db)]: for query column
    c = e*rho + r (rotate(eyes[e], r)) and template j, inner = <a', b'> and
    overlap = |m_a AND m_b| (iris_core.cpp:37-51; pipeline.cpp:78-82, 140-151)."""
    ctx = ctx or default_context()
    dc, dm, d = _stack(db)
    qc, qm, dq = _stack(eyes)
    if db and eyes and d != dq:
        raise ShapeMismatch("template lengths differ")
    d = d or dq
    cols = len(eyes) * rho
    inner = np.zeros((cols, len(db)), np.int32)
    ovl = np.zeros((cols, len(db)), np.int32)
    ctx.check(capi.lib().irl_iris_inner_overlap(ctx.handle, _p(dc), _p(dm), len(db), _p(qc), _p(qm),
                                                len(eyes), rho, d, _p(inner), _p(ovl)))
    return inner, ovl


def match_eyes(db: Sequence[IrisTemplate], eyes: Sequence[IrisTemplate], rho: int, p_int: Interval,
               ctx: Optional[Context] = None, want_scores: bool = False):
    """Per eye e: match_db_reference([rotate(eyes[e], r) for r < rho], db, ., p_int)
    as 1 / 0 / -1 (ZeroOverlap); per-(eye, template) match bits; optional
    scores [cols][n_db] (NaN where the overlap is empty). Does not raise."""
    ctx = ctx or default_context()
    dc, dm, d = _stack(db)
    qc, qm, dq = _stack(eyes)
    if db and eyes and d != dq:
        raise ShapeMismatch("template lengths differ")
    d = d or dq
    bits = np.zeros((len(eyes), len(db)), np.uint8)
    res = np.zeros(len(eyes), np.int32)
    sc = np.zeros((len(eyes) * rho, len(db)), np.float64) if want_scores else None
    st = capi.lib().irl_iris_match(ctx.handle, _p(dc), _p(dm), len(db), _p(qc), _p(qm), len(eyes), rho, d,
                                   float(p_int.lo), float(p_int.hi), _p(bits), _p(res), _p(sc))
    if st not in (capi.IRL_OK, capi.IRL_ERR_ZERO_OVERLAP):
        ctx.check(st)
    return res, bits, sc


def match_db_reference(query: Sequence[IrisTemplate], db: Sequence[IrisTemplate], n_int: Interval,
                       p_int: Interval, ctx: Optional[Context] = None) -> bool:
    """iris::match_db_reference (iris_core.cpp:78-90): True at the first
    (query, entry) score in p_int, ZeroOverlap if an empty overlap comes first
    in that loop order, else False."""
    if not query or not db:
        return False
    res, _, _ = match_eyes(db, query, 1, p_int, ctx)
    for r in res:  # query-major order: the first eye with an event decides
        if r == 1:
            return True
        if r == -1:
            raise ZeroOverlap("mask overlap is empty, score undefined")
    return False


def score(a: IrisTemplate, b: IrisTemplate, ctx: Optional[Context] = None) -> float:
    """iris::score (iris_core.cpp:55-59)."""
    if a.size() != b.size():
        raise ShapeMismatch("template lengths differ")
    inner, ovl = inner_overlap([b], [a], 1, ctx)
    if ovl[0, 0] == 0:
        raise ZeroOverlap("mask overlap is empty, score undefined")
    return float(inner[0, 0]) / float(ovl[0, 0])


class IrisDatabase:
    """Device-resident enrolled templates (irl_iris_db_*): planes built once in
    HBM; each match() moves only the query eyes' bits to the device."""

    def __init__(self, db: Sequence[IrisTemplate], max_cols: int, ctx: Optional[Context] = None):
        import ctypes as C
        self.ctx = ctx or default_context()
        dc, dm, d = _stack(db)
        self.n_db, self.d, self.max_cols = len(db), d, max_cols
        h = C.c_void_p()
        self.ctx.check(capi.lib().irl_iris_db_create(self.ctx.handle, _p(dc), _p(dm), len(db), d, max_cols,
                                                     C.byref(h)))
        self.handle = h

    @classmethod
    def from_packed(cls, code: np.ndarray, mask: np.ndarray, d: int, max_cols: int,
                    ctx: Optional[Context] = None) -> "IrisDatabase":
        import ctypes as C
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        self.n_db, self.d, self.max_cols = code.shape[0], d, max_cols
        h = C.c_void_p()
        self.ctx.check(capi.lib().irl_iris_db_create(self.ctx.handle, _p(code), _p(mask), code.shape[0], d,
                                                     max_cols, C.byref(h)))
        self.handle = h
        return self

    @classmethod
    def from_file(cls, path, max_cols: int, ctx: Optional[Context] = None) -> "IrisDatabase":
        """The enrolled templates straight from the reference's template file
        (save_templates, iris_core.cpp:183-196)."""
        import ctypes as C
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        n, d = C.c_size_t(), C.c_size_t()
        self.ctx.check(capi.lib().irl_iris_db_create_file(self.ctx.handle, str(path).encode(), max_cols, C.byref(h),
                                                          C.byref(n), C.byref(d)))
        self.handle = h
        self.n_db, self.d, self.max_cols = n.value, d.value, max_cols
        return self

    def match_packed(self, q_code, q_mask, n_eyes: int, rho: int, p_int: Interval, want_scores=False,
                     out_bits=None):
        """out_bits: optional C-contiguous uint8 [n_eyes][n_db] array the match bits are
        written into (and returned), so a caller matching batch after batch reuses one
        buffer instead of faulting in fresh pages every call."""
        if out_bits is None:
            bits = np.zeros((n_eyes, self.n_db), np.uint8)
        else:
            bits = out_bits
            if bits.dtype != np.uint8 or bits.shape != (n_eyes, self.n_db) or not bits.flags.c_contiguous:
                raise ValueError("out_bits must be a C-contiguous uint8 array of shape (n_eyes, n_db)")
        res = np.zeros(n_eyes, np.int32)
        sc = np.zeros((n_eyes * rho, self.n_db), np.float64) if want_scores else None
        st = capi.lib().irl_iris_db_match(self.handle, _p(q_code), _p(q_mask), n_eyes, rho, float(p_int.lo),
                                          float(p_int.hi), _p(bits), _p(res), _p(sc))
        if st not in (capi.IRL_OK, capi.IRL_ERR_ZERO_OVERLAP):
            self.ctx.check(st)
        return res, bits, sc

    def match(self, eyes: Sequence[IrisTemplate], rho: int, p_int: Interval, want_scores=False):
        """Same outputs as match_eyes(db, eyes, rho, p_int)."""
        qc, qm, d = _stack(eyes)
        if eyes and d != self.d:
            raise ShapeMismatch("template lengths differ")
        return self.match_packed(qc, qm, len(eyes), rho, p_int, want_scores)

    def fold_packed(self, q_code, q_mask, n_eyes: int, cfg, want_folded: bool = True,
                    want_refolded: Optional[bool] = None, out_folded=None, out_refolded=None):
        """run_alg2's post-CCMM stage against this database (irl_iris_db_fold):
        products and overlaps of the query eyes' rotations as tensor-core GEMMs (FP4), then
        the fold stage (fold.py) on the device. cfg: fold.FoldConfig with
        cfg.d == the template length and n_db == len(db). out_folded / out_refolded:
        optional C-contiguous float64 arrays of the result shapes to write into and
        return (reused across batches; page-locked ones are copied to by DMA directly)."""
        import ctypes as C

        from .fold import FoldResult, _Params, shapes
        if want_refolded is None:
            want_refolded = bool(cfg.fold_chain)
        p = _Params(cfg, n_eyes, self.n_db)
        fshape, rshape = shapes(cfg, n_eyes, self.n_db)

        def out(want, given, shape):
            if not want or cfg.d <= 0:
                return None
            if given is None:
                return np.zeros(shape)
            if given.dtype != np.float64 or given.shape != tuple(shape) or not given.flags.c_contiguous:
                raise ValueError(f"output buffer must be a C-contiguous float64 array of shape {tuple(shape)}")
            return given
        folded = out(want_folded, out_folded, fshape)
        refolded = out(want_refolded, out_refolded, rshape)
        ok = C.c_int32(-1)
        self.ctx.check(capi.lib().irl_iris_db_fold(self.handle, _p(q_code), _p(q_mask), p.ref(),
                                                   _p(folded), _p(refolded), C.byref(ok)))
        return FoldResult(folded, refolded, bool(ok.value))

    def fold(self, eyes: Sequence[IrisTemplate], cfg, want_folded: bool = True,
             want_refolded: Optional[bool] = None):
        qc, qm, d = _stack(eyes)
        if eyes and d != self.d:
            raise ShapeMismatch("pipeline: query template dimension mismatch")
        return self.fold_packed(qc, qm, len(eyes), cfg, want_folded, want_refolded)

    def close(self):
        if getattr(self, "handle", None):
            capi.lib().irl_iris_db_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def save_templates(path, templates: Sequence[IrisTemplate]):
    """The reference's packed template file (iris_core.cpp:183-196): little-endian
    header {magic 0x49524954, version 1, n, d}, then the code plane and the mask
    plane, each n*d bits back to back, bit i of byte j = element 8j + i."""
    n = len(templates)
    d = templates[0].size() if n else 0
    for t in templates:
        if t.size() != d:
            raise ShapeMismatch("all templates must share one length")
    hdr = (0x49524954).to_bytes(4, "little") + (1).to_bytes(4, "little") + n.to_bytes(8, "little") + \
        d.to_bytes(8, "little")
    code = np.concatenate([np.asarray(t.code, np.uint8) for t in templates]) if n else np.zeros(0, np.uint8)
    mask = np.concatenate([np.asarray(t.mask, np.uint8) for t in templates]) if n else np.zeros(0, np.uint8)
    with open(path, "wb") as f:
        f.write(hdr)
        f.write(np.packbits(code, bitorder="little").tobytes())
        f.write(np.packbits(mask, bitorder="little").tobytes())

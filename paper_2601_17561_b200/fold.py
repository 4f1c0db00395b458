"""Alg. 2 fold stage on the B200 (C ABI irl_fold_stage*, csrc/fold.cu).

Mirrors what run_alg2 (reference pipeline.cpp:538-633) does to the score
ciphertexts between the CCMM and the discretization, at message level:
normalize by the mask overlaps (pipe::normalize, :359-371), the degree-7
folding polynomial with the Rot alignment and the group sums
(pipe::fold_group, :391-408), the fold classifier chain (pipe::eval_chain_ct,
:379-389) and the refold across rotation groups (:612-627), plus the
folding-assumption shadow check (:565-590). The outputs equal the messages of
the reference's noise-free emulator bit for bit.

Inputs are the CCMM product and the overlaps in the [c][n_db] layout of
iris.inner_overlap (c = e*rho + r); IrisDatabase.fold runs the whole path
from enrolled templates on the device.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

import numpy as np

from . import capi
from .modmat import Context, default_context

# data/fold_poly_appc.json of the reference: the published folding polynomial
FOLD_POLY_APPC = (0.004105, -0.17351, -2.528271, 24.347349, 124.16155, -412.746212, 376.961251, 106.553952)


@dataclass
class FoldConfig:
    """The PipelineConfig fields the fold stage reads (pipeline.hpp:16-45).
    fold_chain: [(center, coeffs)] -- ClassifierChain::Stage (poly_design.hpp:66-72)."""
    rho: int = 31
    fold_k: int = 16
    d: int = 1024
    fold_poly: Sequence[float] = FOLD_POLY_APPC
    fold_chain: Sequence[Tuple[float, Sequence[float]]] = field(default_factory=list)
    negative: Tuple[float, float] = (-0.25, 0.25)


@dataclass
class FoldResult:
    folded: Optional[np.ndarray]    # [batch][blocks][groups][d] fold_group messages
    refolded: Optional[np.ndarray]  # [batch][blocks][d] refolded messages
    assumption_ok: bool             # PipelineResult::folding_assumption_ok


class _Params:
    """irl_fold_params plus the arrays it points into (kept alive)."""

    def __init__(self, cfg: FoldConfig, batch: int, n_db: int):
        self.fold = np.ascontiguousarray(cfg.fold_poly, np.float64)
        chain = list(cfg.fold_chain)
        self.centers = np.array([float(c) for c, _ in chain] or [0.0], np.float64)
        self.lens = np.array([len(p) for _, p in chain] or [0], np.uintp)
        self.coeffs = np.ascontiguousarray(
            np.concatenate([np.asarray(p, np.float64) for _, p in chain]) if chain else np.zeros(1))
        f64p = C.POINTER(C.c_double)
        self.c = capi.FoldParams(
            batch=batch, rho=cfg.rho, n_db=n_db, d=cfg.d, fold_k=cfg.fold_k,
            fold_coeffs=self.fold.ctypes.data_as(f64p), fold_len=len(self.fold),
            chain_stages=len(chain), chain_centers=self.centers.ctypes.data_as(f64p),
            chain_lens=self.lens.ctypes.data_as(C.POINTER(C.c_size_t)),
            chain_coeffs=self.coeffs.ctypes.data_as(f64p),
            negative_lo=float(cfg.negative[0]), negative_hi=float(cfg.negative[1]))

    def ref(self):
        return C.byref(self.c)


def shapes(cfg: FoldConfig, batch: int, n_db: int):
    blocks = n_db // cfg.d if cfg.d else 0
    groups = -(-cfg.rho // cfg.fold_k) if cfg.fold_k else 0
    return (batch, blocks, groups, cfg.d), (batch, blocks, cfg.d)


def fold_stage(inner: np.ndarray, overlap: np.ndarray, batch: int, cfg: FoldConfig, want_folded: bool = True,
               want_refolded: Optional[bool] = None, ctx: Optional[Context] = None) -> FoldResult:
    """Host buffers: inner / overlap int32 [batch*rho][n_db]. Raises
    ConfigError (PipelineConfig::validate order and messages) and ZeroOverlap
    like the reference's run_alg2. want_refolded defaults to "the chain is
    not empty" (eval_chain_ct rejects an empty chain)."""
    ctx = ctx or default_context()
    if want_refolded is None:
        want_refolded = bool(cfg.fold_chain)
    inner = np.ascontiguousarray(inner, np.int32)
    overlap = np.ascontiguousarray(overlap, np.int32)
    n_db = inner.shape[1]
    p = _Params(cfg, batch, n_db)
    fshape, rshape = shapes(cfg, batch, n_db)
    folded = np.zeros(fshape) if want_folded and cfg.d > 0 else None
    refolded = np.zeros(rshape) if want_refolded and cfg.d > 0 else None
    ok = C.c_int32(-1)
    ctx.check(capi.lib().irl_fold_stage(ctx.handle, p.ref(), capi.ptr(inner), capi.ptr(overlap),
                                        capi.ptr(folded) if folded is not None else None,
                                        capi.ptr(refolded) if refolded is not None else None, C.byref(ok)))
    return FoldResult(folded, refolded, bool(ok.value))


def fold_stage_device(inner, overlap, batch: int, cfg: FoldConfig, folded=None, refolded=None, flags=None,
                      stream=None, ctx: Optional[Context] = None):
    """Device (torch) buffers, stream-ordered. flags: int32[2] device tensor
    OR-ed into ([0] assumption violated, [1] empty overlap); returned."""
    import torch
    ctx = ctx or default_context()
    n_db = inner.shape[1]
    p = _Params(cfg, batch, n_db)
    if flags is None:
        flags = torch.zeros(2, dtype=torch.int32, device=inner.device)
    if stream is None:
        stream = torch.cuda.current_stream(inner.device).cuda_stream
    if not stream:
        stream = 0x1  # torch's default stream is the legacy stream (NULL would mean the context stream)
    ctx.check(capi.lib().irl_fold_stage_device(
        ctx.handle, p.ref(), capi.ptr(inner), capi.ptr(overlap), capi.ptr(folded) if folded is not None else None,
        capi.ptr(refolded) if refolded is not None else None, capi.ptr(flags), C.c_void_p(stream)))
    return flags

"""RGSW-based CCMM engine on the B200.

The encrypted database (MSRLWE-RGSW) is four matrices mod Q:
A1 (N_db x d2), B1 (d1 x d2), A2 (N_db x N_qry), B2 (d1 x N_qry); the query is
Aq (N_qry x d3) and Bq (d2 x d3). The product is two matrices

    out_A = A1 Bq + A2 Aq   (N_db x d3)      -- the shared a-part
    out_B = B1 Bq + B2 Aq   (d1 x d3)        -- one b-part per DB slice

i.e. four PPMMs mod Q. Each part is ONE K-concatenated GEMM
[X1 | X2] [Bq ; Aq] with K = d2 + N_qry, run per RNS modulus as three fused
int8 tensor-core GEMMs. Parts follow the paper's 8-slice layout: part 0 is the
a-part, parts 1..7 are b-part slices of 2^14 templates.

Outputs are residues mod p_i^2, laid out [part][modulus][column n][row m]:
column n of a part is the coefficient vector of the ciphertext(s) that hold
output column n (each ciphertext = N_db consecutive rows of one column, as in
Emulator::ccmm_twin, emulator.cpp:422-446).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import capi
from .modmat import Context, RnsBasis, build_paper_basis, default_context


class CcmmEngine:
    def __init__(self, parts: int, m: int, k: int, max_n: int, basis: Optional[RnsBasis] = None,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.basis = basis or build_paper_basis()
        self.parts, self.M, self.K, self.max_n = parts, m, k, max_n
        self.primes, self.exps = self.basis.arrays()
        self.nmod = len(self.primes)
        h = C.c_void_p()
        self.ctx.check(capi.lib().irl_ccmm_create(
            self.ctx.handle, parts, m, k, max_n, capi.ptr(self.primes, capi.u32p),
            capi.ptr(self.exps, capi.u32p), self.nmod, C.byref(h)))
        self.handle = h

    @property
    def moduli(self):
        return [int(p) ** int(e) for p, e in zip(self.primes, self.exps)]

    @property
    def device_bytes(self) -> int:
        return int(capi.lib().irl_ccmm_device_bytes(self.handle))

    def load_part(self, part: int, residues):
        """residues: [nmod][M][K] uint16 (numpy host array or CUDA torch tensor)."""
        on_dev = hasattr(residues, "data_ptr") and getattr(residues, "is_cuda", False)
        if not on_dev:
            residues = np.ascontiguousarray(residues, np.uint16)
            assert residues.shape == (self.nmod, self.M, self.K)
        self.ctx.check(capi.lib().irl_ccmm_load_part(self.handle, part, capi.ptr(residues), int(on_dev)))

    def load_part_bigint(self, part: int, entries: np.ndarray, width: int):
        """entries: [M][K] fixed-width little-endian integers mod Q."""
        entries = np.ascontiguousarray(entries, np.uint8)
        self.ctx.check(capi.lib().irl_ccmm_load_part_bigint(self.handle, part, capi.ptr(entries, capi.u8p),
                                                            width))

    def load_part_file(self, part: int, path):
        """Stream a part from the reference's BigMatrix file (modmat.cpp:216-231)."""
        self.ctx.check(capi.lib().irl_ccmm_load_part_file(self.handle, part, str(path).encode()))

    def synth_db(self, seed: int, first_part: int = 0):
        """Counter-based synthetic residues, identical to oracle's orc_synth_residue;
        local part g is global part first_part + g."""
        self.ctx.check(capi.lib().irl_ccmm_synth_db(self.handle, seed, first_part))

    def run(self, q_res: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        """End-to-end with host buffers: q_res [nmod][K][N] -> [parts][nmod][N][M]."""
        assert q_res.dtype == np.uint16 and q_res.flags.c_contiguous
        n = q_res.shape[2]
        assert q_res.shape == (self.nmod, self.K, n)
        if out is None:
            out = np.empty((self.parts, self.nmod, n, self.M), np.uint16)
        self.ctx.check(capi.lib().irl_ccmm_run(self.handle, capi.ptr(q_res), n, capi.ptr(out)))
        return out

    def run_device(self, q_res_dev, n: int, out_dev, part0: int = 0, nparts: Optional[int] = None,
                   q_ready: bool = False, stream=None):
        """Device-resident run on torch CUDA tensors; stream-ordered, non-blocking.
        stream: a raw cudaStream_t handle; default = torch's current stream, so
        the run is ordered after the torch ops that filled the inputs."""
        nparts = self.parts - part0 if nparts is None else nparts
        s = C.c_void_p(stream if stream is not None else _torch_stream(self.ctx.device))
        self.ctx.check(capi.lib().irl_ccmm_run_device(
            self.handle, capi.ptr(q_res_dev) if q_res_dev is not None else None, int(q_ready), n,
            part0, nparts, capi.ptr(out_dev) if out_dev is not None else None, s))

    def run_dq(self, q_res_dev, n: int, out: np.ndarray, stream=None) -> np.ndarray:
        """Query on the device (CUDA tensor [nmod][K][n] or None = the staging
        buffer), outputs to host `out` [parts][nmod][n][M] (pinned for speed);
        ordered after `stream` (default: torch's current stream); blocks."""
        assert out.dtype == np.uint16 and out.flags.c_contiguous and out.shape == (self.parts, self.nmod, n, self.M)
        s = C.c_void_p(stream if stream is not None else _torch_stream(self.ctx.device))
        self.ctx.check(capi.lib().irl_ccmm_run_dq(self.handle, capi.ptr(q_res_dev) if q_res_dev is not None else None,
                                                  n, capi.ptr(out), s))
        return out

    def rescale(self, n: int, dst, drop: int, round_: bool = True, part0: int = 0,
                nparts: Optional[int] = None, stream=None):
        """ModDown (f2) of the engine outputs of the last device run: parts
        [part0, part0 + nparts) -> dst [nparts][nmod - drop][n][M] (CUDA tensor)."""
        nparts = self.parts - part0 if nparts is None else nparts
        s = C.c_void_p(stream if stream is not None else _torch_stream(self.ctx.device))
        self.ctx.check(capi.lib().irl_ccmm_rescale(self.handle, n, part0, nparts, drop, int(round_),
                                                   capi.ptr(dst), s))

    # ---- fused a-part exchange (irl_ccmm_alloc_recv / set_mirrors) ----------

    RECV_SLOTS = 2  # IRL_RECV_SLOTS

    def alloc_recv(self, n: int, parts: int = 1):
        """Engine-owned double-buffered receive buffer [2][nmod][n][M] (or
        [2][parts][nmod][n][M] for an a-part spanning `parts` row blocks) for
        the a-part: returns a torch view (int16 bit patterns) and its 64-byte
        CUDA IPC handle. The owner stores step s into slot set_mirror_slot(s % 2)."""
        import torch
        p = C.c_void_p()
        h = (C.c_uint8 * 64)()
        self.ctx.check(capi.lib().irl_ccmm_alloc_recv_parts(self.handle, n, parts, C.byref(p), h))
        shape = (self.RECV_SLOTS,) + ((parts,) if parts > 1 else ()) + (self.nmod, n, self.M)
        view = torch.as_tensor(_CudaArray(p.value, shape, "<i2"), device=f"cuda:{self.ctx.device}")
        return view, bytes(h)

    def set_mirror_parts(self, count: int):
        """Mirror `count` consecutive local parts from the mirrored part on
        (an a-part dealt as several row blocks)."""
        self.ctx.check(capi.lib().irl_ccmm_set_mirror_parts(self.handle, count))

    def synth_part(self, part: int, seed: int, global_part: int, row0: int):
        """Local part `part` = rows [row0, row0 + M) of global part global_part
        of the synthetic database (row-block dealing)."""
        self.ctx.check(capi.lib().irl_ccmm_synth_part(self.handle, part, seed, global_part, row0))

    def set_mirror_slot(self, slot: int):
        """Receive slot of the peers' buffers the next runs store into."""
        self.ctx.check(capi.lib().irl_ccmm_set_mirror_slot(self.handle, slot))

    def set_mirrors(self, part: int, n: int, handles):
        """Store part `part`'s outputs also into the peers' buffers (IPC handles)."""
        buf = (C.c_uint8 * (64 * len(handles)))(*b"".join(handles)) if handles else None
        self.ctx.check(capi.lib().irl_ccmm_set_mirrors(self.handle, part, n, buf, len(handles)))

    def set_mirror_ptrs(self, part: int, n: int, tensors):
        """Same with device tensors of this process (tests)."""
        arr = (C.c_void_p * max(1, len(tensors)))(*[t.data_ptr() for t in tensors])
        self.ctx.check(capi.lib().irl_ccmm_set_mirror_ptrs(self.handle, part, n, arr, len(tensors)))

    @classmethod
    def borrowed(cls, handle, ctx: Context, parts: int, m: int, k: int, max_n: int, basis: RnsBasis):
        """A view of an engine owned elsewhere (a rank of CcmmGroup)."""
        self = cls.__new__(cls)
        self.ctx, self.basis, self.handle, self._borrowed = ctx, basis, handle, True
        self.parts, self.M, self.K, self.max_n = parts, m, k, max_n
        self.primes, self.exps = basis.arrays()
        self.nmod = len(self.primes)
        return self

    def close(self):
        if getattr(self, "handle", None) and not getattr(self, "_borrowed", False):
            capi.lib().irl_ccmm_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CcmmGroup:
    """The CCMM across several devices in one process (irl_ccmm_group_*,
    irl_ccmm_full): one engine per entry of `devices`, parts dealt as
    dist.part_range (the a-part on rank 0), the a-part result stored into every
    other rank by rank 0's PPMM epilogue: through an NVLS multicast address
    (one rank per multicast-capable device) or P2P stores into each peer."""

    def __init__(self, devices, parts: int, m: int, k: int, max_n: int, basis: Optional[RnsBasis] = None):
        self.basis = basis or build_paper_basis()
        self.primes, self.exps = self.basis.arrays()
        self.nmod = len(self.primes)
        self.devices = list(devices)
        self.parts, self.M, self.K, self.max_n = parts, m, k, max_n
        devs = (C.c_int * len(self.devices))(*self.devices)
        h = C.c_void_p()
        st = capi.lib().irl_ccmm_group_create(devs, len(self.devices), parts, m, k, max_n,
                                              capi.ptr(self.primes, capi.u32p), capi.ptr(self.exps, capi.u32p),
                                              self.nmod, C.byref(h))
        if st != capi.IRL_OK:
            from .modmat import _STATUS_EXC, DeviceError
            raise _STATUS_EXC.get(st, DeviceError)(f"irl_ccmm_group_create: {capi.lib().irl_status_string(st).decode()}")
        self.handle = h
        self.ctx = Context.borrowed(capi.lib().irl_ccmm_group_ctx(h, 0), self.devices[0])

    def engine(self, rank: int):
        """(engine view, first global part, part count) of a rank."""
        e, first, count = C.c_void_p(), C.c_size_t(), C.c_size_t()
        self.ctx.check(capi.lib().irl_ccmm_group_engine(self.handle, rank, C.byref(e), C.byref(first),
                                                        C.byref(count)))
        ctx = Context.borrowed(capi.lib().irl_ccmm_group_ctx(self.handle, rank), self.devices[rank])
        eng = CcmmEngine.borrowed(e, ctx, count.value, self.M, self.K, self.max_n, self.basis)
        return eng, first.value, count.value

    def synth_db(self, seed: int):
        for r in range(len(self.devices)):
            eng, first, _ = self.engine(r)
            eng.synth_db(seed, first_part=first)

    def set_exchange(self, mode: int):
        """capi.IRL_EXCHANGE_AUTO / _P2P / _MULTICAST / _COPY (irl_ccmm_group_set_exchange)."""
        self.ctx.check(capi.lib().irl_ccmm_group_set_exchange(self.handle, mode))

    def set_query_shard(self, mode: int):
        """-1 auto, 0 every rank copies the whole query, 1 sharded host copies plus a
        peer all-gather (irl_ccmm_group_set_query_shard)."""
        self.ctx.check(capi.lib().irl_ccmm_group_set_query_shard(self.handle, mode))

    def run(self, q_res: np.ndarray, out: Optional[np.ndarray] = None):
        """q_res [nmod][K][n] -> (out [parts][nmod][n][M], per-rank device
        pointers of the a-part result, the IRL_EXCHANGE_* mode used)."""
        assert q_res.dtype == np.uint16 and q_res.flags.c_contiguous
        n = q_res.shape[2]
        if out is None:
            out = np.empty((self.parts, self.nmod, n, self.M), np.uint16)
        ptrs = (C.c_void_p * len(self.devices))()
        mode = C.c_int(-1)
        self.ctx.check(capi.lib().irl_ccmm_full(self.handle, capi.ptr(q_res), n, capi.ptr(out), ptrs,
                                                C.byref(mode)))
        return out, [p for p in ptrs], mode.value

    def a_part(self, rank: int, ptr: int, n: int):
        """torch view (int16 bit patterns) of a rank's copy of the a-part result."""
        import torch
        return torch.as_tensor(_CudaArray(ptr, (self.nmod, n, self.M), "<i2"), device=f"cuda:{self.devices[rank]}")

    def close(self):
        if getattr(self, "handle", None):
            capi.lib().irl_ccmm_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _torch_stream(device: int) -> int:
    """torch's current stream on `device` as a cudaStream_t handle (the legacy
    default stream is handle 0 in torch, cudaStreamLegacy = 0x1 for the ABI,
    where NULL means the context's own stream)."""
    import torch
    h = torch.cuda.current_stream(device).cuda_stream
    return h if h else 0x1


def synth_query(seed: int, k: int, n: int, moduli, stream: int = 0xFF) -> np.ndarray:
    """Synthetic query residues [nmod][K][N] from the shared counter generator."""
    out = np.empty((len(moduli), k, n), np.uint16)
    L = capi.lib()
    for i, m in enumerate(moduli):
        L.irl_synth_residues_host(seed, stream, i, 0, k, 0, n, m, capi.ptr(out[i], capi.u16p))
    return out


class _CudaArray:
    """Minimal __cuda_array_interface__ view of engine-owned device memory."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def staging_tensors(engine: CcmmEngine, n: int):
    """torch views (int16 bit patterns of the uint16 residues) of the engine's
    device staging buffers: query residues [nmod][K][n] and outputs
    [parts][nmod][n][M]. Zero-copy; valid while the engine lives."""
    import torch
    qp, op = C.c_void_p(), C.c_void_p()
    engine.ctx.check(capi.lib().irl_ccmm_buffers(engine.handle, C.byref(qp), C.byref(op)))
    dev = f"cuda:{engine.ctx.device}"
    q = torch.as_tensor(_CudaArray(qp.value, (engine.nmod, engine.K, n), "<i2"), device=dev)
    o = torch.as_tensor(_CudaArray(op.value, (engine.parts, engine.nmod, n, engine.M), "<i2"), device=dev)
    return q, o


# ---------------------------------------------------------------------------
# Caller drop-in: Emulator::ccmm_twin (reference emulator.hpp:85-97, 135-140;
# emulator.cpp:389-447) with the product computed by the PPMM engine.
# ---------------------------------------------------------------------------

from dataclasses import dataclass


@dataclass
class CcmmSpec:
    d1: int = 0
    d2: int = 0
    d3: int = 0
    n_db: int = 0
    n_qry: int = 0
    db_modulus_bits: float = 0.0
    qry_modulus_bits: float = 0.0
    scale_bits: float = 0.0
    out_level: int = 0
    out_encoding: str = "coeff"   # "coeff" | "slot"
    out_ci: bool = False


@dataclass
class CcmmOutput:
    """d1*d3/n_db ciphertexts in ccmm_twin's order (column-major over (c, b)):
    messages[k] is the n_db-slot message of output ciphertext k."""
    messages: np.ndarray           # [d3 * d1 / n_db][n_db] float64
    level: int
    encoding: str
    ci: bool
    log_ring_degree: int
    scale_bits: float


def ccmm_twin(spec: CcmmSpec, db, qry, top_level: int, ctx: Optional[Context] = None) -> CcmmOutput:
    """Exact product db (d1 x d2) . qry (d2 x d3) packed as ccmm_twin packs it,
    with its shape / modulus-budget checks and exception types."""
    ctx = ctx or default_context()
    db = np.ascontiguousarray(db, np.float64).ravel()
    qry = np.ascontiguousarray(qry, np.float64).ravel()
    if spec.d1 > 0 and spec.d2 > 0 and spec.d3 > 0 and spec.n_db > 0 and spec.n_qry > 0 and \
            spec.d1 % spec.n_db == 0 and spec.d2 % spec.n_qry == 0 and \
            (db.size != spec.d1 * spec.d2 or qry.size != spec.d2 * spec.d3):
        from .modmat import ShapeMismatch
        raise ShapeMismatch("ccmm: matrix buffer sizes do not match dimensions")
    out = np.empty(max(spec.d1 * spec.d3, 1), np.float64)
    dp = C.POINTER(C.c_double)
    ctx.check(capi.lib().irl_ccmm_twin(
        ctx.handle, spec.d1, spec.d2, spec.d3, spec.n_db, spec.n_qry, spec.db_modulus_bits,
        spec.qry_modulus_bits, spec.scale_bits, spec.out_level, top_level,
        int(spec.out_encoding == "slot"), int(spec.out_ci), db.ctypes.data_as(dp), qry.ctypes.data_as(dp),
        out.ctypes.data_as(dp)))
    return CcmmOutput(messages=out.reshape(-1, spec.n_db), level=spec.out_level, encoding=spec.out_encoding,
                      ci=spec.out_ci, log_ring_degree=int(spec.n_db).bit_length() - 1,
                      scale_bits=spec.scale_bits)

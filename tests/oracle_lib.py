"""ctypes bindings for the TEST oracle (oracle/libirl_oracle.so) and, when it
was built in this container, the unmodified reference (oracle/_ref/libirl_ref.so).

Test infrastructure only: the product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "libirl_oracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libirl_ref.so"

M64 = (1 << 64) - 1

u8p = C.POINTER(C.c_uint8)
i8p = C.POINTER(C.c_int8)
u16p = C.POINTER(C.c_uint16)
i32p = C.POINTER(C.c_int32)
u32p = C.POINTER(C.c_uint32)
i64p = C.POINTER(C.c_int64)
sz = C.c_size_t


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


_oracle = None
_ref = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not ORACLE_SO.exists():
            subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)
        lib = C.CDLL(str(ORACLE_SO))
        lib.orc_primes_in_range.restype = sz
        lib.orc_primes_in_range.argtypes = [C.c_uint32, C.c_uint32, u32p, sz]
        lib.orc_paper_basis.restype = sz
        lib.orc_paper_basis.argtypes = [u32p, u32p, sz]
        lib.orc_log2_Q.restype = C.c_double
        lib.orc_log2_Q.argtypes = [u32p, u32p, sz]
        lib.orc_max_int8_rns_capacity.restype = C.c_double
        lib.orc_pure_rns_plane_count.restype = sz
        lib.orc_basis_Q_bytes.restype = sz
        lib.orc_basis_Q_bytes.argtypes = [u32p, u32p, sz, u8p, sz]
        lib.orc_digit_decompose.argtypes = [i32p, sz, C.c_uint32, i32p, i32p]
        lib.orc_digit_recompose.argtypes = [i32p, i32p, sz, C.c_uint32, i32p]
        lib.orc_small_gemm.argtypes = [i32p, i32p, i32p, sz, sz, sz, i64p]
        lib.orc_gemm_mod_psq.argtypes = [i32p, i32p, i32p, sz, sz, sz, C.c_uint32]
        lib.orc_gemm_mod_Q.argtypes = [u8p, u8p, u8p, sz, sz, sz, sz, u32p, u32p, sz]
        lib.orc_oracle_gemm_mod_Q.argtypes = [u8p, u8p, u8p, sz, sz, sz, sz, u32p, u32p, sz]
        lib.orc_ppmm_rows_direct.argtypes = [u16p, sz, u16p, sz, u32p, sz, sz, sz, C.c_uint32, u16p]
        lib.orc_ccmm_twin_product.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), sz, sz, sz,
                                              C.POINTER(C.c_double)]
        lib.orc_synth_residue.restype = C.c_uint32
        lib.orc_synth_residue.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]
        lib.orc_iris_inner_overlap.argtypes = [u8p, u8p, sz, u8p, u8p, sz, sz, sz, i32p, i32p]
        lib.orc_synth_block.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.c_uint32, C.c_uint32, C.c_uint32, u16p]
        f64p = C.POINTER(C.c_double)
        lib.orc_ps_execute.restype = C.c_double
        lib.orc_ps_execute.argtypes = [f64p, sz, C.c_double]
        lib.orc_fold_stage.argtypes = [sz, sz, sz, sz, sz, f64p, sz, sz, f64p, C.POINTER(sz), f64p,
                                       C.c_double, C.c_double, i32p, i32p, f64p, f64p, i32p]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(str(REF_SO))
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_paper_basis.restype = sz
        lib.ref_paper_basis.argtypes = [u32p, u32p, sz]
        lib.ref_digit_planes.restype = sz
        lib.ref_log2_Q.restype = C.c_double
        lib.ref_max_int8_rns_capacity.restype = C.c_double
        lib.ref_pure_rns_plane_count.restype = sz
        lib.ref_paper_Q_bytes.restype = sz
        lib.ref_paper_Q_bytes.argtypes = [u8p, sz]
        lib.ref_digit_decompose.argtypes = [i32p, sz, sz, C.c_uint32, i32p, i32p]
        lib.ref_digit_recompose.argtypes = [i32p, i32p, sz, sz, C.c_uint32, i32p]
        lib.ref_small_gemm.argtypes = [i32p, i32p, i32p, sz, sz, sz]
        lib.ref_gemm_mod_psq.argtypes = [i32p, i32p, i32p, sz, sz, sz, C.c_uint32]
        lib.ref_gemm_mod_psq_batch.argtypes = [C.POINTER(i32p), C.POINTER(i32p), C.POINTER(i32p), u32p,
                                               sz, sz, sz, sz, C.c_int]
        lib.ref_gemm_mod_Q.argtypes = [u8p, u8p, u8p, sz, sz, sz, sz, u32p, u32p, sz]
        lib.ref_oracle_gemm_mod_Q.argtypes = [u8p, u8p, u8p, sz, sz, sz, sz, u32p, u32p, sz]
        lib.ref_crit2_next.argtypes = [C.POINTER(sz), C.POINTER(sz), C.POINTER(sz), u8p, u8p, sz]
        lib.ref_random_big.argtypes = [C.c_uint64, sz, sz, sz, u8p, sz]
        lib.ref_save_load_roundtrip.argtypes = [C.c_char_p, u8p, sz, sz, sz, u8p]
        lib.ref_synth_masked.argtypes = [sz, sz, C.c_double, C.c_uint64, i8p]
        lib.ref_synth_masked_rotated.argtypes = [sz, sz, C.c_double, C.c_uint64, sz, i8p]
        lib.ref_synth_templates.argtypes = [sz, sz, C.c_double, C.c_uint64, u8p, u8p]
        f64p = C.POINTER(C.c_double)
        lib.ref_iris_scores.argtypes = [u8p, u8p, sz, u8p, u8p, sz, sz, f64p]
        lib.ref_iris_rotate.argtypes = [u8p, u8p, sz, sz, u8p, u8p]
        lib.ref_save_templates.argtypes = [C.c_char_p, u8p, u8p, sz, sz]
        lib.ref_match_db_reference.argtypes = [u8p, u8p, sz, u8p, u8p, sz, sz, C.c_double, C.c_double,
                                               C.c_double, C.c_double, C.POINTER(C.c_int)]
        lib.ref_ps_execute.argtypes = [f64p, sz, C.c_double, f64p]
        lib.ref_ccmm_twin.argtypes = [C.c_long, C.c_long, C.c_long, C.c_long, C.c_long, C.c_double, C.c_double,
                                      C.c_double, C.c_int, C.c_int, C.c_int, f64p, f64p, f64p, C.POINTER(C.c_int)]
        lib.ref_fold_stage.argtypes = [sz, sz, sz, sz, sz, f64p, sz, sz, f64p, C.POINTER(sz), f64p, i32p, i32p,
                                       f64p, f64p]
        lib.ref_alg2_assumption.argtypes = [u8p, u8p, sz, u8p, u8p, sz, sz, sz, sz, f64p, sz, sz, f64p,
                                            C.POINTER(sz), f64p, C.c_double, C.c_double, C.POINTER(C.c_int)]
        _ref = lib
    return _ref


PIPE_SO = {"ref": ROOT / "oracle" / "_ref" / "libirl_pipe_ref.so",
           "b200": ROOT / "oracle" / "_ref" / "libirl_pipe_b200.so"}
_pipe = {}


def pipe_available() -> bool:
    return all(p.exists() for p in PIPE_SO.values())


def pipe(kind: str) -> C.CDLL:
    """The reference's end-to-end pipeline (oracle/pipe_capi.cpp over the
    unmodified emulator/pipeline sources): kind "ref" = stock ccmm_twin,
    "b200" = ccmm_twin's product from the B200 engine (link-time wrap)."""
    if kind not in _pipe:
        lib = C.CDLL(str(PIPE_SO[kind]))
        lib.pipe_last_error.restype = C.c_char_p
        lib.pipe_planted_small.argtypes = [i64p]
        lib.pipe_instances.argtypes = [C.c_int, C.c_int, C.c_long, C.c_int, C.c_uint64, C.POINTER(C.c_double), sz,
                                       i64p, sz]
        lib.irl_hook_digest.restype = C.c_uint64
        lib.irl_hook_calls.restype = C.c_long
        lib.irl_hook_slots.restype = C.c_long
        _pipe[kind] = lib
    return _pipe[kind]


# --------------------------------------------------------------------------
# Basis and big-integer helpers (Python ints)
# --------------------------------------------------------------------------

def paper_basis():
    p = np.zeros(64, np.uint32)
    e = np.zeros(64, np.uint32)
    n = oracle().orc_paper_basis(ptr(p, u32p), ptr(e, u32p), 64)
    return p[:n].copy(), e[:n].copy()


def basis_Q(primes, exps) -> int:
    q = 1
    for p, e in zip(primes, exps):
        q *= int(p) ** int(e)
    return q


def width_of(Q: int) -> int:
    return (Q.bit_length() + 7) // 8


def ints_to_le(vals, width: int) -> np.ndarray:
    out = np.zeros((len(vals), width), np.uint8)
    for i, v in enumerate(vals):
        out[i] = np.frombuffer(int(v).to_bytes(width, "little"), np.uint8)
    return out


def le_to_ints(arr: np.ndarray, width: int):
    flat = np.ascontiguousarray(arr).reshape(-1, width)
    return [int.from_bytes(bytes(row), "little") for row in flat]


class MT19937_64:
    """std::mt19937_64 (used by the reference tests' generators)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & M64
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & M64
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & M64


def random_big(rng: MT19937_64, rows: int, cols: int, Q: int):
    """tests/test_modmat.cpp:12-22: six 32-bit words, big-endian concat, mod Q."""
    out = []
    for _ in range(rows * cols):
        x = 0
        for _w in range(6):
            x = (x << 32) + (rng() & 0xFFFFFFFF)
        out.append(x % Q)
    return out


def schoolbook_mod(a, b, m, k, n, Q):
    """Arbitrary-precision reference product (oracle_gemm_mod_Q semantics)."""
    out = []
    for i in range(m):
        for j in range(n):
            out.append(sum(a[i * k + t] * b[t * n + j] for t in range(k)) % Q)
    return out


# --------------------------------------------------------------------------
# Oracle wrappers (numpy in/out)
# --------------------------------------------------------------------------

def orc_gemm_mod_psq(a: np.ndarray, b: np.ndarray, p: int):
    a = np.ascontiguousarray(a, np.int32)
    b = np.ascontiguousarray(b, np.int32)
    m, k = a.shape
    k2, n = b.shape
    assert k == k2
    c = np.zeros((m, n), np.int32)
    st = oracle().orc_gemm_mod_psq(ptr(a, i32p), ptr(b, i32p), ptr(c, i32p), m, k, n, p)
    return st, c


def orc_gemm_mod_Q(a_le, b_le, m, k, n, width, primes, exps):
    c = np.zeros((m * n, width), np.uint8)
    st = oracle().orc_gemm_mod_Q(ptr(a_le, u8p), ptr(b_le, u8p), ptr(c, u8p), m, k, n, width,
                                 ptr(primes, u32p), ptr(exps, u32p), len(primes))
    return st, c


def orc_ccmm_twin_product(db: np.ndarray, qry: np.ndarray) -> np.ndarray:
    """emulator.cpp:411-421 restated in C: db (d1 x d2) . qry (d2 x d3) in the
    reference's operation order, returned in message order [d3][d1]."""
    db = np.ascontiguousarray(db, np.float64)
    qry = np.ascontiguousarray(qry, np.float64)
    d1, d2 = db.shape
    d3 = qry.shape[1]
    out = np.zeros((d3, d1), np.float64)
    f64p = C.POINTER(C.c_double)
    oracle().orc_ccmm_twin_product(db.ctypes.data_as(f64p), qry.ctypes.data_as(f64p), d1, d2, d3,
                                   out.ctypes.data_as(f64p))
    return out


def ref_ccmm_twin(db: np.ndarray, qry: np.ndarray, n_db: int, n_qry: int, db_bits=100.0, q_bits=50.0,
                  scale=23.0, out_level=0, out_slot=0, out_ci=0):
    """The reference's Emulator::ccmm_twin (noise-free default emulator):
    (status, messages [d3][d1] real parts, chain top level)."""
    db = np.ascontiguousarray(db, np.float64)
    qry = np.ascontiguousarray(qry, np.float64)
    d1, d2 = db.shape
    d3 = qry.shape[1]
    out = np.zeros((d3, d1), np.float64)
    top = C.c_int(0)
    f64p = C.POINTER(C.c_double)
    st = ref().ref_ccmm_twin(d1, d2, d3, n_db, n_qry, db_bits, q_bits, scale, out_level, out_slot, out_ci,
                             db.ctypes.data_as(f64p), qry.ctypes.data_as(f64p), out.ctypes.data_as(f64p),
                             C.byref(top))
    return st, out, top.value


def twin_doubles(d1, d2, d3, seed):
    """Non-integer operands exercising the rounding order: mixed magnitudes,
    exact zeros and negative zeros in the database, an inf in the query."""
    rng = np.random.default_rng(seed)
    db = rng.standard_normal((d1, d2)) * np.exp2(rng.integers(-30, 30, (d1, d2)))
    db[rng.random((d1, d2)) < 0.2] = 0.0
    db[rng.random((d1, d2)) < 0.05] = -0.0
    qry = rng.standard_normal((d2, d3)) * np.exp2(rng.integers(-20, 20, (d2, d3)))
    return db, qry


def synth_block(seed, stream, plane, row0, nrows, col0, ncols, m):
    out = np.zeros((nrows, ncols), np.uint16)
    oracle().orc_synth_block(seed, stream, plane, row0, nrows, col0, ncols, m, ptr(out, u16p))
    return out


def ppmm_rows_direct(a: np.ndarray, bt: np.ndarray, rows, m: int):
    """a [R][K] uint16, bt [N][K] uint16 -> out [len(rows)][N] = a[rows] bt^T mod m."""
    a = np.ascontiguousarray(a, np.uint16)
    bt = np.ascontiguousarray(bt, np.uint16)
    rows = np.ascontiguousarray(rows, np.uint32)
    N, K = bt.shape
    out = np.zeros((len(rows), N), np.uint16)
    oracle().orc_ppmm_rows_direct(ptr(a, u16p), a.shape[1], ptr(bt, u16p), K, ptr(rows, u32p),
                                  len(rows), N, K, m, ptr(out, u16p))
    return out


# --------------------------------------------------------------------------
# Plaintext iris scoring (oracle restatement + reference wrappers)
# --------------------------------------------------------------------------

def iris_inner_overlap(db_code, db_mask, q_code, q_mask, rho):
    """Oracle: int32 inner, overlap [n_eyes*rho][n_db] (iris_core.cpp:37-51)."""
    db_code, db_mask = (np.ascontiguousarray(x, np.uint8) for x in (db_code, db_mask))
    q_code, q_mask = (np.ascontiguousarray(x, np.uint8) for x in (q_code, q_mask))
    n_db, d = db_code.shape
    ne = q_code.shape[0]
    inner = np.zeros((ne * rho, n_db), np.int32)
    ovl = np.zeros((ne * rho, n_db), np.int32)
    oracle().orc_iris_inner_overlap(ptr(db_code, u8p), ptr(db_mask, u8p), n_db, ptr(q_code, u8p),
                                    ptr(q_mask, u8p), ne, rho, d, ptr(inner, i32p), ptr(ovl, i32p))
    return inner, ovl


def ref_synth_templates(n, d, density, seed):
    code = np.zeros((n, d), np.uint8)
    mask = np.zeros((n, d), np.uint8)
    st = ref().ref_synth_templates(n, d, density, seed, ptr(code, u8p), ptr(mask, u8p))
    assert st == 0
    return code, mask


def ref_rotate(code, mask, r):
    d = code.shape[0]
    oc, om = np.zeros(d, np.uint8), np.zeros(d, np.uint8)
    code, mask = np.ascontiguousarray(code, np.uint8), np.ascontiguousarray(mask, np.uint8)
    ref().ref_iris_rotate(ptr(code, u8p), ptr(mask, u8p), d, r, ptr(oc, u8p), ptr(om, u8p))
    return oc, om


def ref_scores(q_code, q_mask, db_code, db_mask):
    nq, d = q_code.shape
    n_db = db_code.shape[0]
    out = np.zeros((nq, n_db), np.float64)
    args = [np.ascontiguousarray(x, np.uint8) for x in (q_code, q_mask, db_code, db_mask)]
    st = ref().ref_iris_scores(ptr(args[0], u8p), ptr(args[1], u8p), nq, ptr(args[2], u8p), ptr(args[3], u8p),
                               n_db, d, out.ctypes.data_as(C.POINTER(C.c_double)))
    assert st == 0
    return out


def ref_match(q_code, q_mask, db_code, db_mask, p_lo, p_hi, n_lo=-1.0, n_hi=0.1):
    """-> 1 / 0, or -1 for ZeroOverlap (status 11)."""
    nq, d = q_code.shape
    n_db = db_code.shape[0]
    args = [np.ascontiguousarray(x, np.uint8) for x in (q_code, q_mask, db_code, db_mask)]
    out = C.c_int(0)
    st = ref().ref_match_db_reference(ptr(args[0], u8p), ptr(args[1], u8p), nq, ptr(args[2], u8p),
                                      ptr(args[3], u8p), n_db, d, n_lo, n_hi, p_lo, p_hi, C.byref(out))
    if st == 11:
        return -1
    assert st == 0, st
    return out.value


def rescale_oracle(res, moduli, drop, round_):
    """ModDown restated with Python integers (test-only, small cases): CRT lift
    of each element (modmat.cpp:178-193), y = floor((x + h) / Delta) mod Q/Delta
    with h = floor(Delta/2) if round_ else 0, residues mod the kept moduli.
    res: [nmod][count] ints."""
    moduli = [int(m) for m in moduli]
    Q = 1
    for m in moduli:
        Q *= m
    delta = 1
    for m in moduli[len(moduli) - drop:]:
        delta *= m
    q2 = Q // delta
    h = delta // 2 if round_ else 0
    coef = []
    for m in moduli:
        qi = Q // m
        coef.append(qi * pow(qi % m, -1, m))
    out = np.zeros((len(moduli) - drop, res.shape[1]), np.uint16)
    for e in range(res.shape[1]):
        x = sum(int(res[i, e]) % m * c for i, (m, c) in enumerate(zip(moduli, coef))) % Q
        y = ((x + h) % Q) // delta % q2
        for i, m in enumerate(moduli[:len(moduli) - drop]):
            out[i, e] = y % m
    return out


# --------------------------------------------------------------------------
# Alg. 2 fold stage (pipeline.cpp:359-408, 538-633)
# --------------------------------------------------------------------------

# data/fold_poly_appc.json: the published degree-7 folding polynomial
FOLD_POLY_APPC = np.array([0.004105, -0.17351, -2.528271, 24.347349, 124.16155, -412.746212,
                           376.961251, 106.553952])


def _compose(p, q):
    """Coefficients of p(q(y)) (ascending), numpy polynomial arithmetic."""
    from numpy.polynomial import polynomial as P
    out = np.array([0.0])
    for c in p[::-1]:
        out = P.polyadd(P.polymul(out, q), [c])
    return out


def fold_chain_for_tests(kind: str = "step"):
    """A stand-in fold classifier chain (list of (center, coeffs)): smooth sign
    approximants f3 = (3z - z^3)/2, f5 = (15z - 10z^3 + 3z^5)/8 and
    f7 = (35z - 35z^3 + 21z^5 - 5z^7)/16, composed and scaled, ending in a
    [0, 1] step. The reference designs its chains offline (compose_classifier,
    poly_design.cpp); any coefficients exercise the same evaluation path.
    "step": degrees 7, 21, 3; "wide": degrees 15, 31, 3."""
    f3 = np.array([0.0, 1.5, 0.0, -0.5])
    f5 = np.array([0.0, 15, 0, -10, 0, 3]) / 8.0
    f7 = np.array([0.0, 35, 0, -35, 0, 21, 0, -5]) / 16.0
    scale = lambda c, a: c * a ** np.arange(len(c))  # noqa: E731
    step = np.array([0.5, 0.75, 0.0, -0.25])
    if kind == "wide":
        f27 = _compose(f3, _compose(f3, f3))
        f31 = np.r_[f27, 0.0, 0.0, 0.0, 1e-9]
        return [(0.365, scale(_compose(f3, f5), 1 / 1024)), (0.0, f31), (0.0, step)]
    return [(0.365, scale(f7, 1 / 256)), (0.0, _compose(f7, f3)), (0.0, step)]


def _chain_arrays(chain):
    centers = np.array([c for c, _ in chain], np.float64)
    lens = np.array([len(p) for _, p in chain], np.uintp)
    coeffs = np.concatenate([np.asarray(p, np.float64) for _, p in chain]) if chain else np.zeros(1)
    return centers, lens, np.ascontiguousarray(coeffs)


def orc_fold(inner, overlap, batch, rho, d, fold_k, fold_c, chain, neg, want_folded=True, want_refold=True):
    """Oracle restatement (oracle/irl_oracle.c orc_fold_stage); returns
    (status, folded, refolded, assumption_ok)."""
    f64p = C.POINTER(C.c_double)
    n_db = inner.shape[1]
    blocks, groups = n_db // d, -(-rho // fold_k)
    folded = np.zeros(batch * blocks * groups * d) if want_folded else None
    refold = np.zeros(batch * blocks * d) if want_refold else None
    fc = np.ascontiguousarray(fold_c, np.float64) if len(fold_c) else np.zeros(1)
    centers, lens, cc = _chain_arrays(chain)
    ok = C.c_int32(-1)
    st = oracle().orc_fold_stage(batch, rho, n_db, d, fold_k, ptr(fc, f64p), len(fold_c), len(chain),
                                 ptr(centers, f64p), lens.ctypes.data_as(C.POINTER(sz)), ptr(cc, f64p),
                                 neg[0], neg[1], ptr(np.ascontiguousarray(inner, np.int32), i32p),
                                 ptr(np.ascontiguousarray(overlap, np.int32), i32p),
                                 ptr(folded, f64p) if folded is not None else None,
                                 ptr(refold, f64p) if refold is not None else None, C.byref(ok))
    return st, folded, refold, ok.value


def ref_fold(inner, overlap, batch, rho, d, fold_k, fold_c, chain, want_refold=True):
    """The reference's own pipe::normalize / fold_group / eval_chain_ct
    (oracle/_ref); returns (status, folded, refolded)."""
    f64p = C.POINTER(C.c_double)
    n_db = inner.shape[1]
    blocks, groups = n_db // d, -(-rho // fold_k)
    folded = np.zeros(batch * blocks * groups * d)
    refold = np.zeros(batch * blocks * d) if want_refold else None
    fc = np.ascontiguousarray(fold_c, np.float64)
    centers, lens, cc = _chain_arrays(chain)
    st = ref().ref_fold_stage(batch, rho, n_db, d, fold_k, ptr(fc, f64p), len(fc), len(chain),
                              ptr(centers, f64p), lens.ctypes.data_as(C.POINTER(sz)), ptr(cc, f64p),
                              ptr(np.ascontiguousarray(inner, np.int32), i32p),
                              ptr(np.ascontiguousarray(overlap, np.int32), i32p), ptr(folded, f64p),
                              ptr(refold, f64p) if refold is not None else None)
    return st, folded, refold


def ref_alg2_flag(q_code, q_mask, db_code, db_mask, rho, fold_k, fold_c, chain, neg):
    """run_alg2's folding_assumption_ok from the reference itself."""
    f64p = C.POINTER(C.c_double)
    fc = np.ascontiguousarray(fold_c, np.float64)
    centers, lens, cc = _chain_arrays(chain)
    ok = C.c_int(-1)
    st = ref().ref_alg2_assumption(ptr(q_code, u8p), ptr(q_mask, u8p), q_code.shape[0], ptr(db_code, u8p),
                                   ptr(db_mask, u8p), db_code.shape[0], db_code.shape[1], rho, fold_k,
                                   ptr(fc, f64p), len(fc), len(chain), ptr(centers, f64p),
                                   lens.ctypes.data_as(C.POINTER(sz)), ptr(cc, f64p), neg[0], neg[1],
                                   C.byref(ok))
    assert st == 0, ref().ref_last_error()
    return ok.value


def orc_inner_overlap(db_code, db_mask, q_code, q_mask, rho):
    n_db, d = db_code.shape
    eyes = q_code.shape[0]
    inner = np.zeros((eyes * rho, n_db), np.int32)
    ovl = np.zeros_like(inner)
    oracle().orc_iris_inner_overlap(ptr(db_code, u8p), ptr(db_mask, u8p), n_db, ptr(q_code, u8p),
                                    ptr(q_mask, u8p), eyes, rho, d, ptr(inner, i32p), ptr(ovl, i32p))
    return inner, ovl

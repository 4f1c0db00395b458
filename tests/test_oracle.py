"""Pins the CPU oracle (oracle/irl_oracle.c) against the reference's own
known-answer tests (tests/golden/, generated from the unmodified reference by
oracle/gen_golden.py) and, when oracle/_ref was built here, against the
reference library directly on fresh random inputs. CPU only."""
import hashlib
import json

import numpy as np
import pytest

import oracle_lib as ol

GOLD = json.loads((ol.ROOT / "tests" / "golden" / "modmat_kats.json").read_text())
P, E = ol.paper_basis()
Q = ol.basis_Q(P, E)
W = ol.width_of(Q)


def test_paper_basis_matches_reference():
    # test_modmat.cpp:26-43
    g = GOLD["basis"]
    assert P.tolist() == g["primes"] and E.tolist() == g["exps"]
    assert len(P) == 24 and 2 * len(P) == g["digit_planes"] == 48
    assert int(min(int(p) ** 2 for p in P)) == 16129
    log2q = ol.oracle().orc_log2_Q(ol.ptr(P, ol.u32p), ol.ptr(E, ol.u32p), len(P))
    assert log2q == pytest.approx(g["log2_Q"], rel=1e-9)
    assert log2q == pytest.approx(sum(2 * np.log2(float(p)) for p in P), rel=1e-9)
    cap = ol.oracle().orc_max_int8_rns_capacity()
    assert log2q > cap and log2q < 362.0
    assert Q == int(g["Q_hex"], 16) and W == g["width"] == 46
    buf = np.zeros(64, np.uint8)
    w = ol.oracle().orc_basis_Q_bytes(ol.ptr(P, ol.u32p), ol.ptr(E, ol.u32p), len(P), ol.ptr(buf, ol.u8p), 64)
    assert w == W and int.from_bytes(bytes(buf[:w]), "little") == Q


def test_capacity_and_plane_economy():
    # test_modmat.cpp:45-53, acceptance criterion 3 (acceptance.cpp:124-136)
    g = GOLD["basis"]
    cap = ol.oracle().orc_max_int8_rns_capacity()
    assert cap == pytest.approx(g["capacity"], abs=1e-9)
    assert abs(cap - 354.83) <= 0.05
    assert ol.oracle().orc_pure_rns_plane_count() == g["pure_planes"] == 53
    assert g["digit_planes"] < g["pure_planes"]
    primes = np.zeros(64, np.uint32)
    n = ol.oracle().orc_primes_in_range(3, 253, ol.ptr(primes, ol.u32p), 64)
    assert primes[0] == 3 and 17 in primes[:n].tolist()


@pytest.mark.parametrize("case", GOLD["digit_decompose"], ids=lambda c: f"p{c['p']}_{c['rows']}x{c['cols']}")
def test_digit_decompose_golden(case):
    # test_modmat.cpp:55-76
    a = np.array(case["input"], np.int32)
    d0 = np.zeros_like(a)
    d1 = np.zeros_like(a)
    st = ol.oracle().orc_digit_decompose(ol.ptr(a, ol.i32p), a.size, case["p"], ol.ptr(d0, ol.i32p), ol.ptr(d1, ol.i32p))
    assert st == case["status"]
    if st == 0:
        assert d0.tolist() == case["d0"] and d1.tolist() == case["d1"]
        half = (case["p"] - 1) // 2
        assert np.abs(d0).max(initial=0) <= max(half, case["p"] - half - 1)
        back = np.zeros_like(a)
        ol.oracle().orc_digit_recompose(ol.ptr(d0, ol.i32p), ol.ptr(d1, ol.i32p), a.size, case["p"], ol.ptr(back, ol.i32p))
        p2 = case["p"] ** 2
        assert ((back.astype(np.int64) - a.astype(np.int64)) % p2 == 0).all()


def _mat(case, key, rows, cols):
    if case.get(key) is not None:
        return np.array(case[key], np.int32).reshape(rows, cols)
    return np.full((rows, cols), case[key + "_fill"], np.int32)


@pytest.mark.parametrize("case", GOLD["small_gemm"], ids=lambda c: c["note"])
def test_small_gemm_golden(case):
    # test_modmat.cpp:79-95
    m, k, n = case["m"], case["k"], case["n"]
    a = _mat(case, "a", m, k)
    b = _mat(case, "b", k, n)
    c = np.zeros((m, n), np.int32)
    bound = np.zeros(1, np.int64)
    st = ol.oracle().orc_small_gemm(ol.ptr(a, ol.i32p), ol.ptr(b, ol.i32p), ol.ptr(c, ol.i32p), m, k, n, ol.ptr(bound, ol.i64p))
    assert st == case["status"]
    if st == 0:
        assert c.ravel().tolist() == case["c"]
    else:
        assert str(int(bound[0])) in case["message"]


@pytest.mark.parametrize("case", GOLD["gemm_mod_psq"], ids=lambda c: c["note"])
def test_gemm_mod_psq_golden(case):
    # test_modmat.cpp:97-123
    a = np.array(case["a"], np.int32).reshape(case["m"], case["k"])
    b = np.array(case["b"], np.int32).reshape(case["k"], case["n"])
    st, c = ol.orc_gemm_mod_psq(a, b, case["p"])
    assert st == case["status"]
    if st == 0:
        assert c.ravel().tolist() == case["c"]


def test_gemm_mod_psq_kat_values():
    # 300 * 500 mod 127^2 = 4839 (test_modmat.cpp:104-106)
    st, c = ol.orc_gemm_mod_psq(np.array([[300]]), np.array([[500]]), 127)
    assert st == 0 and int(c[0, 0]) == 150000 % 16129 == 4839


def test_gemm_mod_Q_seed7_stream():
    # test_modmat.cpp:125-145: identity, zero, 5 x random 32^3 from mt19937_64(7)
    rng = ol.MT19937_64(7)
    bq = ol.random_big(rng, 8, 8, Q)
    ident = [1 if i == j else 0 for i in range(8) for j in range(8)]
    inputs = [(ident, bq, 8, 8, 8), ([0] * 64, bq, 8, 8, 8)]
    for _ in range(5):
        inputs.append((ol.random_big(rng, 32, 32, Q), ol.random_big(rng, 32, 32, Q), 32, 32, 32))
    for (a, b, m, k, n), gold in zip(inputs, GOLD["gemm_mod_Q_seed7"]):
        st, c = ol.orc_gemm_mod_Q(ol.ints_to_le(a, W), ol.ints_to_le(b, W), m, k, n, W, P, E)
        assert st == 0
        assert hashlib.sha256(c.tobytes()).hexdigest() == gold["sha256"], gold["name"]
    got = ol.le_to_ints(ol.orc_gemm_mod_Q(ol.ints_to_le(ident, W), ol.ints_to_le(bq, W), 8, 8, 8, W, P, E)[1], W)
    assert got == bq


def test_acceptance_criterion2_instances():
    # acceptance.cpp:96-120: exact equality with the reference on its own stream
    data = np.load(ol.ROOT / "tests" / "golden" / "crit2_instances.npz")
    idx = sorted({k.split("_")[0] for k in data.files})
    assert len(idx) >= 8
    for i in idx:
        a, b, c = data[i + "_a"], data[i + "_b"], data[i + "_c"]
        m, k, _ = a.shape
        n = b.shape[1]
        st, got = ol.orc_gemm_mod_Q(np.ascontiguousarray(a), np.ascontiguousarray(b), m, k, n, W, P, E)
        assert st == 0 and (got.reshape(c.shape) == c).all(), i
        got2 = np.zeros_like(got)
        ol.oracle().orc_oracle_gemm_mod_Q(ol.ptr(np.ascontiguousarray(a), ol.u8p), ol.ptr(np.ascontiguousarray(b), ol.u8p),
                                          ol.ptr(got2, ol.u8p), m, k, n, W, ol.ptr(P, ol.u32p), ol.ptr(E, ol.u32p), len(P))
        assert (got2.reshape(c.shape) == c).all(), i


DIG = json.loads((ol.ROOT / "tests" / "golden" / "c1_crit2_digests.json").read_text())


def test_oracle_c1_rows_match_reference_digest():
    # BASELINE configs[0] (p = 127, 256 x 4096 . 4096 x 4096): the oracle's
    # first 16 output rows equal the reference's (digest from oracle/_ref)
    g = DIG["c1"]
    m = 127 * 127
    a = ol.synth_block(1, 0, 0, 0, 16, 0, 4096, m).astype(np.int32)
    b = ol.synth_block(1, 1, 0, 0, 4096, 0, 4096, m).astype(np.int32)
    assert hashlib.sha256(b.tobytes()).hexdigest() == g["b_sha256"]
    st, c = ol.orc_gemm_mod_psq(a, b, 127)
    assert st == 0 and c[0, :8].tolist() == g["c_head"]
    assert hashlib.sha256(c.tobytes()).hexdigest() == g["c_rows16_sha256"]


@pytest.mark.skipif(not ol.ref_available(), reason="oracle/_ref not built")
def test_oracle_crit2_stream_matches_reference_digests():
    # acceptance.cpp:96-120: the oracle's gemm_mod_Q on every 10th instance of
    # the reference's own 1000-instance stream equals the reference's digest
    R = ol.ref()
    R.ref_crit2_reset()
    abuf = np.zeros((64 * 64, W), np.uint8)
    bbuf = np.zeros((64 * 64, W), np.uint8)
    for idx, (m, k, n, in_dig, out_dig) in enumerate(DIG["crit2"]["instances"]):
        m_, k_, n_ = ol.sz(), ol.sz(), ol.sz()
        R.ref_crit2_next(m_, k_, n_, ol.ptr(abuf, ol.u8p), ol.ptr(bbuf, ol.u8p), W)
        assert (m_.value, k_.value, n_.value) == (m, k, n)
        if idx % 10:
            continue
        a, b = abuf[: m * k].copy(), bbuf[: k * n].copy()
        assert hashlib.sha256(a.tobytes() + b.tobytes()).hexdigest()[:32] == in_dig
        st, c = ol.orc_gemm_mod_Q(a, b, m, k, n, W, P, E)
        assert st == 0 and hashlib.sha256(c.tobytes()).hexdigest()[:32] == out_dig, idx


@pytest.mark.skipif(not ol.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [1, 2])
def test_oracle_ccmm_twin_product_equals_reference_on_doubles(seed):
    # emulator.cpp:411-421 on arbitrary doubles (fractions, 2^+-30 magnitude
    # spread, +-0 database entries, an inf in the query): the C restatement
    # reproduces the reference's messages bit for bit
    d1, d2, d3, n_db = 64, 48, 6, 16
    db, qry = ol.twin_doubles(d1, d2, d3, seed)
    qry[3, 2] = np.inf             # +-inf in output column 2
    db[0, 0], qry[0, 4] = np.inf, 0.0  # inf * 0 = NaN in output (0, 4)
    st, want, _ = ol.ref_ccmm_twin(db, qry, n_db, 16)
    assert st == 0
    got = ol.orc_ccmm_twin_product(db, qry)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert np.isnan(got[4, 0]) and np.isinf(got[2]).any()


def test_ccmm_composition_on_iris_kat():
    # Our RGSW composition restatement on the reference's own iris inputs
    # (synth_db/to_masked/rotate): per-prime products of ternary matrices,
    # CRT-lifted and centred, equal the exact integer product that
    # Emulator::ccmm_twin computes (emulator.cpp:411-421).
    data = np.load(ol.ROOT / "tests" / "golden" / "iris_kat.npz")
    db, qry, prod = data["db"], data["qry"], data["prod"]
    sub_m, sub_n = 24, 10
    a = [int(v) % Q for v in db[:sub_m].astype(np.int64).ravel()]
    b = [int(v) % Q for v in qry[:, :sub_n].astype(np.int64).ravel()]
    st, c = ol.orc_gemm_mod_Q(ol.ints_to_le(a, W), ol.ints_to_le(b, W), sub_m, db.shape[1], sub_n, W, P, E)
    assert st == 0
    vals = [v - Q if v > Q // 2 else v for v in ol.le_to_ints(c, W)]
    assert np.array(vals).reshape(sub_m, sub_n).tolist() == prod[:sub_m, :sub_n].tolist()


def test_ccmm_twin_kat_product():
    # test_emulator.cpp:215-245: (4x3)(3x2) -> columns (11,3,3,5), (14,4,6,6)
    g = GOLD["ccmm_twin"]
    db = np.array(g["db"]).reshape(g["d1"], g["d2"])
    qry = np.array(g["qry"]).reshape(g["d2"], g["d3"])
    prod = db @ qry
    assert prod[:, 0].tolist() == g["col0"] and prod[:, 1].tolist() == g["col1"]
    assert g["d1"] // g["n_db"] * g["d3"] == g["outputs"]


def test_synth_generator_is_counter_based_and_uniform():
    a = ol.synth_block(1, 3, 5, 100, 64, 7, 128, 16129)
    b = ol.synth_block(1, 3, 5, 100 + 10, 4, 7 + 20, 8, 16129)
    assert (a[10:14, 20:28] == b).all()
    assert a.max() < 16129
    big = ol.synth_block(9, 0, 0, 0, 256, 0, 1024, 63001).astype(np.float64)
    assert abs(big.mean() / 63000 - 0.5) < 0.01


def test_ppmm_direct_equals_digit_path():
    rng = np.random.default_rng(3)
    p = 251
    a = rng.integers(0, p * p, (12, 300)).astype(np.int32)
    b = rng.integers(0, p * p, (300, 9)).astype(np.int32)
    st, c = ol.orc_gemm_mod_psq(a, b, p)
    assert st == 0
    d = ol.ppmm_rows_direct(a.astype(np.uint16), np.ascontiguousarray(b.T.astype(np.uint16)), np.arange(12), p * p)
    assert (d.astype(np.int32) == c).all()


ref_only = pytest.mark.skipif(not ol.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


@ref_only
@pytest.mark.parametrize("seed", range(4))
def test_oracle_equals_reference_gemm_mod_psq(seed):
    rng = np.random.default_rng(100 + seed)
    m, k, n = rng.integers(1, 40, 3)
    p = int(rng.choice(P))
    a = rng.integers(-2**31, 2**31, (m, k), dtype=np.int64).astype(np.int32)
    b = rng.integers(-2**31, 2**31, (k, n), dtype=np.int64).astype(np.int32)
    st, c = ol.orc_gemm_mod_psq(a, b, p)
    cr = np.zeros_like(c)
    str_ = ol.ref().ref_gemm_mod_psq(ol.ptr(a, ol.i32p), ol.ptr(b, ol.i32p), ol.ptr(cr, ol.i32p), m, k, n, p)
    assert st == str_ == 0 and (c == cr).all()


@ref_only
def test_oracle_equals_reference_gemm_mod_Q_odd_basis():
    # a non-paper basis with e = 1 moduli exercises the small_gemm branch (:177-178)
    primes = np.array([3, 5, 7, 11, 13], np.uint32)
    exps = np.array([2, 1, 2, 1, 1], np.uint32)
    q = ol.basis_Q(primes, exps)
    w = ol.width_of(q)
    rng = np.random.default_rng(7)
    m, k, n = 5, 6, 4
    a = [int(x) % q for x in rng.integers(0, 2**62, m * k)]
    b = [int(x) % q for x in rng.integers(0, 2**62, k * n)]
    al, bl = ol.ints_to_le(a, w), ol.ints_to_le(b, w)
    st, c = ol.orc_gemm_mod_Q(al, bl, m, k, n, w, primes, exps)
    cr = np.zeros_like(c)
    str_ = ol.ref().ref_gemm_mod_Q(ol.ptr(al, ol.u8p), ol.ptr(bl, ol.u8p), ol.ptr(cr, ol.u8p), m, k, n, w,
                                   ol.ptr(primes, ol.u32p), ol.ptr(exps, ol.u32p), len(primes))
    assert st == str_ == 0 and (c == cr).all()
    assert ol.le_to_ints(c, w) == ol.schoolbook_mod(a, b, m, k, n, q)


@ref_only
def test_oracle_equals_reference_not_coprime():
    primes = np.array([3, 3], np.uint32)
    exps = np.array([1, 1], np.uint32)
    al = ol.ints_to_le([1, 2], 1)
    bl = ol.ints_to_le([1, 2], 1)
    st, _ = ol.orc_gemm_mod_Q(al, bl, 1, 2, 1, 1, primes, exps)
    cr = np.zeros((1, 1), np.uint8)
    str_ = ol.ref().ref_gemm_mod_Q(ol.ptr(al, ol.u8p), ol.ptr(bl, ol.u8p), ol.ptr(cr, ol.u8p), 1, 2, 1, 1,
                                   ol.ptr(primes, ol.u32p), ol.ptr(exps, ol.u32p), 2)
    assert st == str_ == 4


def test_rescale_oracle_bruteforce():
    # the f2 ModDown restatement against exhaustive search on a tiny basis
    moduli = [7, 9, 11, 13]
    Q = 7 * 9 * 11 * 13
    xs = np.arange(0, Q, 37)
    res = np.array([[x % m for x in xs] for m in moduli])
    for drop in (1, 2):
        delta = int(np.prod(moduli[len(moduli) - drop:]))
        for rnd in (0, 1):
            got = ol.rescale_oracle(res, moduli, drop, rnd)
            for e, x in enumerate(xs):
                y = ((int(x) + (delta // 2 if rnd else 0)) % Q) // delta
                assert [y % m for m in moduli[:len(moduli) - drop]] == got[:, e].tolist()

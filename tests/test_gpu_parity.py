"""GPU parity suite: the B200 engine (through its C ABI) against the pinned
CPU oracle and the reference's golden vectors. Bit-exact everywhere (integer
work). Run on a B200: pytest -m gpu."""
import hashlib
import json

import numpy as np
import pytest

import oracle_lib as ol

pytestmark = pytest.mark.gpu

GOLD = json.loads((ol.ROOT / "tests" / "golden" / "modmat_kats.json").read_text())


@pytest.fixture(scope="module")
def mm():
    from paper_2601_17561_b200 import modmat
    modmat.default_context()
    return modmat


@pytest.fixture(scope="module")
def basis(mm):
    return mm.build_paper_basis()


# ---------------------------------------------------------------- KATs -------

@pytest.mark.parametrize("case", GOLD["digit_decompose"], ids=lambda c: f"p{c['p']}_{c['rows']}x{c['cols']}")
def test_digit_decompose_golden(mm, case):
    a = np.array(case["input"], np.int32).reshape(case["rows"], case["cols"])
    if case["status"] == 2:
        with pytest.raises(mm.ModulusTooLarge, match="digit base must be < 2\\^8"):
            mm.digit_decompose(a, case["p"])
        return
    d = mm.digit_decompose(a, case["p"])
    assert d.m0.ravel().tolist() == case["d0"] and d.m1.ravel().tolist() == case["d1"]
    back = mm.digit_recompose(d)
    ref = np.zeros_like(back)
    ol.oracle().orc_digit_recompose(ol.ptr(d.m0, ol.i32p), ol.ptr(d.m1, ol.i32p), a.size, case["p"],
                                    ol.ptr(ref, ol.i32p))
    assert (back == ref).all()


@pytest.mark.parametrize("case", GOLD["small_gemm"], ids=lambda c: c["note"])
def test_small_gemm_golden(mm, case):
    m, k, n = case["m"], case["k"], case["n"]
    a = np.array(case["a"], np.int32).reshape(m, k) if case["a"] is not None else np.full((m, k), case["a_fill"], np.int32)
    b = np.array(case["b"], np.int32).reshape(k, n) if case["b"] is not None else np.full((k, n), case["b_fill"], np.int32)
    if case["status"] == 3:
        with pytest.raises(mm.AccumulationOverflowRisk) as ei:
            mm.small_gemm(a, b)
        assert str(ei.value) == case["message"]
        return
    assert mm.small_gemm(a, b).ravel().tolist() == case["c"]


@pytest.mark.parametrize("case", GOLD["gemm_mod_psq"], ids=lambda c: c["note"])
def test_gemm_mod_psq_golden(mm, case):
    a = np.array(case["a"], np.int32).reshape(case["m"], case["k"])
    b = np.array(case["b"], np.int32).reshape(case["k"], case["n"])
    if case["status"] == 2:
        with pytest.raises(mm.ModulusTooLarge):
            mm.gemm_mod_psq(a, b, case["p"])
        return
    assert mm.gemm_mod_psq(a, b, case["p"]).ravel().tolist() == case["c"]


def test_gemm_mod_Q_seed7_stream(mm, basis):
    # test_modmat.cpp:125-145 through the GPU residue/PPMM/CRT path
    Q, W = basis.Q, basis.width()
    rng = ol.MT19937_64(7)
    bq = ol.random_big(rng, 8, 8, Q)
    ident = [1 if i == j else 0 for i in range(8) for j in range(8)]
    inputs = [(ident, bq, 8, 8, 8), ([0] * 64, bq, 8, 8, 8)]
    for _ in range(5):
        inputs.append((ol.random_big(rng, 32, 32, Q), ol.random_big(rng, 32, 32, Q), 32, 32, 32))
    for (a, b, m, k, n), gold in zip(inputs, GOLD["gemm_mod_Q_seed7"]):
        c = mm.gemm_mod_Q_le(ol.ints_to_le(a, W), ol.ints_to_le(b, W), m, k, n, W, basis)
        assert hashlib.sha256(c.tobytes()).hexdigest() == gold["sha256"], gold["name"]
    got = mm.gemm_mod_Q(mm.BigMatrix.identity(8), mm.BigMatrix(8, 8, bq), basis)
    assert got.a == bq


def test_acceptance_criterion2_instances(mm, basis):
    data = np.load(ol.ROOT / "tests" / "golden" / "crit2_instances.npz")
    for i in sorted({k.split("_")[0] for k in data.files}):
        a, b, c = data[i + "_a"], data[i + "_b"], data[i + "_c"]
        m, k, _ = a.shape
        n = b.shape[1]
        got = mm.gemm_mod_Q_le(a, b, m, k, n, basis.width(), basis)
        assert (got.reshape(c.shape) == c).all(), i


def test_gemm_mod_Q_odd_basis_and_errors(mm):
    b = mm.RnsBasis([mm.Modulus(3, 2), mm.Modulus(5, 1), mm.Modulus(7, 2), mm.Modulus(11, 1), mm.Modulus(13, 1)])
    for md in b.moduli:
        b.Q *= md.value()
    rng = np.random.default_rng(7)
    m, k, n = 5, 6, 4
    A = mm.BigMatrix(m, k, [int(x) % b.Q for x in rng.integers(0, 2**62, m * k)])
    B = mm.BigMatrix(k, n, [int(x) % b.Q for x in rng.integers(0, 2**62, k * n)])
    assert mm.gemm_mod_Q(A, B, b).a == ol.schoolbook_mod(A.a, B.a, m, k, n, b.Q)
    bad = mm.RnsBasis([mm.Modulus(3, 1), mm.Modulus(3, 1)], 9)
    with pytest.raises(mm.Error, match="CRT basis is not coprime"):
        mm.gemm_mod_Q(mm.BigMatrix(1, 2, [1, 2]), mm.BigMatrix(2, 1, [1, 2]), bad)
    with pytest.raises(mm.ShapeMismatch):
        mm.gemm_mod_Q(mm.BigMatrix(2, 3), mm.BigMatrix(2, 3), b)


# ------------------------------------------------------ random parity -------

@pytest.mark.parametrize("p,m,k,n", [(127, 1, 1, 1), (251, 37, 515, 29), (149, 256, 4096, 256),
                                     (251, 300, 1000, 200), (3, 16, 64, 16), (254, 40, 129, 33)])
def test_gemm_mod_psq_random_vs_oracle(mm, p, m, k, n):
    rng = np.random.default_rng(p * 1000 + m)
    a = rng.integers(-2**31, 2**31, (m, k), dtype=np.int64).astype(np.int32)
    b = rng.integers(-2**31, 2**31, (k, n), dtype=np.int64).astype(np.int32)
    st, ref = ol.orc_gemm_mod_psq(a, b, p)
    assert st == 0
    assert (mm.gemm_mod_psq(a, b, p) == ref).all()


def test_gemm_mod_psq_k_chunked_accumulation(mm):
    # K * 2 * 125^2 > 2^31 > K * 125^2: the reference accepts it (each small_gemm
    # is in range); the fused A0B1 + A1B0 accumulator must be K-chunked.
    p, m, k, n = 251, 8, 70000, 8
    rng = np.random.default_rng(1)
    a = rng.integers(0, p * p, (m, k)).astype(np.int32)
    b = rng.integers(0, p * p, (k, n)).astype(np.int32)
    st, ref = ol.orc_gemm_mod_psq(a, b, p)
    assert st == 0
    assert (mm.gemm_mod_psq(a, b, p) == ref).all()


def test_overflow_risk_matches_reference(mm):
    k = 1 << 18
    a = np.full((1, k), 125 + 251 * 125, np.int32)  # both digits = 125 at p = 251
    b = a.T.copy()
    st, _ = ol.orc_gemm_mod_psq(a, b, 251)
    assert st == 3
    with pytest.raises(mm.AccumulationOverflowRisk, match="K\\*\\|A\\|\\*\\|B\\|"):
        mm.gemm_mod_psq(a, b, 251)


def test_empty_shapes(mm):
    assert mm.gemm_mod_psq(np.zeros((0, 5), np.int32), np.zeros((5, 3), np.int32), 127).shape == (0, 3)
    assert (mm.gemm_mod_psq(np.zeros((2, 0), np.int32), np.zeros((0, 3), np.int32), 127) == 0).all()
    assert mm.small_gemm(np.zeros((3, 0), np.int32), np.zeros((0, 2), np.int32)).tolist() == [[0, 0]] * 3


# -------------------------------------------------------------- CCMM -------

def _oracle_part(seed, part, i, rows, K, q_i_T, m):
    a = ol.synth_block(seed, part, i, 0, max(rows) + 1, 0, K, m)
    return ol.ppmm_rows_direct(a, q_i_T, rows, m)


def _check_ccmm(eng, seed, q, out, rows):
    from paper_2601_17561_b200.ccmm import CcmmEngine  # noqa
    for part in range(eng.parts):
        for i, m in enumerate(eng.moduli):
            qt = np.ascontiguousarray(q[i].T)
            want = _oracle_part(seed, part, i, rows, eng.K, qt, m)
            got = out[part, i][:, rows].T
            assert (got == want).all(), (part, i)


def test_ccmm_small_all_rows():
    from paper_2601_17561_b200.ccmm import CcmmEngine, synth_query
    eng = CcmmEngine(parts=3, m=300, k=1000, max_n=70)
    eng.synth_db(seed=1)
    q = synth_query(2, eng.K, 70, eng.moduli)
    out = eng.run(q)
    _check_ccmm(eng, 1, q, out, np.arange(300, dtype=np.uint32))


def test_ccmm_load_part_equals_synth():
    from paper_2601_17561_b200.ccmm import CcmmEngine, synth_query
    eng = CcmmEngine(parts=2, m=260, k=700, max_n=64)
    eng.synth_db(seed=5)
    q = synth_query(6, eng.K, 64, eng.moduli)
    want = eng.run(q)
    eng2 = CcmmEngine(parts=2, m=260, k=700, max_n=64)
    for part in range(2):
        res = np.stack([ol.synth_block(5, part, i, 0, 260, 0, 700, m) for i, m in enumerate(eng.moduli)])
        eng2.load_part(part, res)
    assert (eng2.run(q) == want).all()


@pytest.mark.parametrize("max_n,n", [(256, 600), (100, 333), (64, 64)])
def test_ccmm_column_chunked_run(max_n, n):
    # query batches wider than the engine's staging capacity (c5: 256 eyes)
    # stream through it in column chunks; result identical to one wide engine
    from paper_2601_17561_b200.ccmm import CcmmEngine, synth_query
    eng = CcmmEngine(parts=2, m=280, k=900, max_n=max_n)
    eng.synth_db(seed=3)
    q = synth_query(4, eng.K, n, eng.moduli)
    out = eng.run(q)
    wide = CcmmEngine(parts=2, m=280, k=900, max_n=n)
    wide.synth_db(seed=3)
    assert (wide.run(q) == out).all()
    _check_ccmm(eng, 3, q, out, np.array([0, 5, 279], np.uint32))


@pytest.mark.slow
def test_ccmm_slice_shape_sampled_rows():
    # c3 slice geometry (N_db = 2^14, K = d2 + N_qry = 24576, N = 32 x 31 = 992),
    # two parts; rows sampled (each output row depends on one DB row only).
    from paper_2601_17561_b200.ccmm import CcmmEngine, synth_query
    eng = CcmmEngine(parts=2, m=1 << 14, k=24576, max_n=992)
    eng.synth_db(seed=1)
    q = synth_query(2, eng.K, 992, eng.moduli)
    out = eng.run(q)
    rows = np.array([0, 1, 255, 256, 8191, 12345, 16383], np.uint32)
    _check_ccmm(eng, 1, q, out, rows)


def test_ccmm_iris_kat_exact_product(mm, basis):
    # Reference iris inputs (synth_db + to_masked + rotate): the GPU CCMM
    # residues, CRT-lifted and centred, reproduce ccmm_twin's exact product.
    from paper_2601_17561_b200.ccmm import CcmmEngine
    data = np.load(ol.ROOT / "tests" / "golden" / "iris_kat.npz")
    db, qry, prod = data["db"].astype(np.int64), data["qry"].astype(np.int64), data["prod"]
    n_db, d = db.shape
    n = qry.shape[1]
    eng = CcmmEngine(parts=1, m=n_db, k=d, max_n=n)
    mods = eng.moduli
    eng.load_part(0, np.stack([(db % m).astype(np.uint16) for m in mods]))
    out = eng.run(np.ascontiguousarray(np.stack([(qry % m).astype(np.uint16) for m in mods])))
    # CRT lift through the engine's own device kernel (irl_crt_lift) via gemm_mod_Q:
    # here on host with Python ints as an independent check.
    Q = basis.Q
    res = out[0]  # [nmod][n][m]
    for (r, c) in [(0, 0), (5, 17), (n_db - 1, n - 1), (40, 31)]:
        x = 0
        for i, m in enumerate(mods):
            qi = Q // m
            x += qi * ((int(res[i, c, r]) * pow(qi, -1, m)) % m)
        x %= Q
        v = x - Q if x > Q // 2 else x
        assert v == int(prod[r, c])
    # and all entries, mod one modulus, against the exact product
    for i, m in enumerate(mods):
        assert (res[i].T.astype(np.int64) == prod % m).all()


def test_launch_counter_and_native_path(mm):
    ctx = mm.default_context()
    before = ctx.launches
    mm.gemm_mod_psq(np.eye(4, dtype=np.int32), np.eye(4, dtype=np.int32), 127)
    assert ctx.launches > before


# ------------------------------------------------ caller drop-in (f1) ------

def _spec(**kw):
    from paper_2601_17561_b200.ccmm import CcmmSpec
    s = CcmmSpec(d1=4, d2=3, d3=2, n_db=2, n_qry=3, qry_modulus_bits=36.0, scale_bits=23.0,
                 db_modulus_bits=2 * 36.0 - 23.0)
    for k, v in kw.items():
        setattr(s, k, v)
    return s


def test_ccmm_twin_kat_and_errors(mm):
    # test_emulator.cpp:215-270 through the GPU product
    from paper_2601_17561_b200.ccmm import ccmm_twin
    g = GOLD["ccmm_twin"]
    out = ccmm_twin(_spec(), g["db"], g["qry"], top_level=9)
    assert out.messages.shape == (g["outputs"], 2)
    assert out.messages[0].tolist() == [11.0, 3.0] and out.messages[1].tolist() == [3.0, 5.0]
    assert out.messages[2].tolist() == [14.0, 4.0] and out.messages[3][1] == 6.0
    assert out.encoding == "coeff" and out.level == 0
    with pytest.raises(mm.ModulusBudget):
        ccmm_twin(_spec(db_modulus_bits=36.0), g["db"], g["qry"], top_level=9)
    with pytest.raises(mm.ModulusBudget):
        ccmm_twin(_spec(out_level=99), g["db"], g["qry"], top_level=9)
    with pytest.raises(mm.ShapeMismatch):
        ccmm_twin(_spec(out_encoding="slot"), g["db"], g["qry"], top_level=9)
    with pytest.raises(mm.ShapeMismatch):
        ccmm_twin(_spec(d1=5), g["db"], g["qry"], top_level=9)
    raised = ccmm_twin(_spec(out_level=5, out_encoding="slot", out_ci=True), g["db"], g["qry"], top_level=9)
    assert raised.level == 5 and raised.encoding == "slot" and raised.ci and raised.messages[0][0] == 11.0


def test_ccmm_twin_pipeline_sizes_exact():
    # acceptance criteria 6/7 geometry (acceptance.cpp:197-217): n_db=4096,
    # d=1024, batch 4 x rho 31, ternary iris values -> exact product
    from paper_2601_17561_b200.ccmm import ccmm_twin
    rng = np.random.default_rng(11)
    d1, d2, d3 = 4096, 1024, 124
    db = rng.integers(-1, 2, (d1, d2)).astype(np.float64)
    qry = rng.integers(-1, 2, (d2, d3)).astype(np.float64)
    spec = _spec(d1=d1, d2=d2, d3=d3, n_db=d2, n_qry=d2)
    out = ccmm_twin(spec, db, qry, top_level=9)
    prod = (db.astype(np.int64) @ qry.astype(np.int64))
    want = prod.T.reshape(d3, d1 // d2, d2).reshape(-1, d2)  # ct(c, b).message[i] = prod[(b n_db + i), c]
    assert (out.messages == want).all()


@pytest.mark.parametrize("basis_kind", ["paper", "mixed"])
@pytest.mark.parametrize("k,n", [(300, 64), (130, 992), (77, 70), (5, 8)])
def test_split_cols_u16_all_paths(basis_kind, k, n):
    # The query split (irl_split_cols_u16): vectorised kernel (N % 8 == 0; odd
    # p^2 bases take the folded-centring fast path, others the general one)
    # and the scalar kernel; raw uint16 inputs over the full 16-bit range so
    # the reduction mod m is exercised. Digits follow digit_decompose
    # (modmat.cpp:86-106); e = 1 moduli keep one centred digit.
    import ctypes as C
    import torch
    from paper_2601_17561_b200 import capi
    from paper_2601_17561_b200.modmat import default_context
    if basis_kind == "paper":
        primes, exps = ol.paper_basis()
    else:
        primes = np.array([2, 2, 3, 251, 127, 5], np.uint32)
        exps = np.array([1, 2, 2, 1, 2, 2], np.uint32)
    nmod = len(primes)
    rng = np.random.default_rng(k * 1000 + n)
    res = rng.integers(0, 65536, (nmod, k, n), dtype=np.uint32).astype(np.uint16)
    ldk = (k + 15) // 16 * 16
    dres = torch.from_numpy(res.view(np.int16)).cuda()
    planes = torch.full((nmod, 2, n, ldk), 77, dtype=torch.int8, device="cuda")
    ctx = default_context()
    ctx.check(capi.lib().irl_split_cols_u16(ctx.handle, C.c_void_p(dres.data_ptr()), n, k * n, k, n,
                                            capi.ptr(primes, capi.u32p), capi.ptr(exps, capi.u32p), nmod,
                                            C.c_void_p(planes.data_ptr()), ldk, None))
    torch.cuda.synchronize()
    got = planes.cpu().numpy()
    for i in range(nmod):
        p, e = int(primes[i]), int(exps[i])
        x = res[i].astype(np.int64).T  # [n][k]
        half = (p - 1) // 2
        if e == 2:
            d0 = np.zeros(x.shape, np.int32)
            d1 = np.zeros(x.shape, np.int32)
            flat = np.ascontiguousarray(x.reshape(-1).astype(np.int32))
            a0 = np.zeros_like(flat)
            a1 = np.zeros_like(flat)
            assert ol.oracle().orc_digit_decompose(ol.ptr(flat, ol.i32p), flat.size, p, ol.ptr(a0, ol.i32p),
                                                   ol.ptr(a1, ol.i32p)) == 0
            d0, d1 = a0.reshape(x.shape), a1.reshape(x.shape)
        else:
            a = x % p
            d0 = np.where(a > half, a - p, a)
            d1 = np.zeros_like(d0)
        assert (got[i, 0, :, :k] == d0).all(), (basis_kind, i)
        assert (got[i, 1, :, :k] == d1).all(), (basis_kind, i)
        assert (got[i, :, :, k:] == 0).all()


@pytest.mark.parametrize("count", [777, 800])  # scalar path / vectorised path
@pytest.mark.parametrize("drop,round_", [(1, 0), (1, 1), (2, 1), (3, 0), (3, 1)])
def test_rescale_residues_vs_bigint(drop, round_, count):
    # f2: ModDown by the product of the last `drop` moduli, exact against
    # Python big integers (CRT lift, floor / round division, re-reduction)
    import ctypes as C
    import torch
    from paper_2601_17561_b200 import capi
    from paper_2601_17561_b200.modmat import default_context
    primes, exps = ol.paper_basis()
    moduli = [int(p) ** int(e) for p, e in zip(primes, exps)]
    nmod = len(moduli)
    rng = np.random.default_rng(drop * 10 + round_)
    res = np.stack([rng.integers(0, m, count) for m in moduli]).astype(np.uint16)
    res[:, 0] = 0                                         # x = 0
    res[:, 1] = [(m - 1) for m in moduli]                 # x = Q - 1 (wraps when rounding)
    res[:, 2] = [65535 for m in moduli]                   # unreduced inputs
    want = ol.rescale_oracle(res, moduli, drop, round_)
    din = torch.from_numpy(res.view(np.int16)).cuda()
    dout = torch.zeros((nmod - drop, count), dtype=torch.int16, device="cuda")
    ctx = default_context()
    ctx.check(capi.lib().irl_rescale_residues(ctx.handle, C.c_void_p(din.data_ptr()), count, count,
                                              capi.ptr(primes, capi.u32p), capi.ptr(exps, capi.u32p), nmod, drop,
                                              round_, C.c_void_p(dout.data_ptr()), count, None))
    torch.cuda.synchronize()
    assert (dout.cpu().numpy().view(np.uint16) == want).all()


def test_ccmm_rescale_matches_bigint():
    # f2 on the engine: ModDown of real CCMM outputs (drop 3, rounding)
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query
    eng = CcmmEngine(parts=2, m=300, k=500, max_n=40)
    eng.synth_db(seed=9)
    q = synth_query(3, eng.K, 40, eng.moduli)
    qd, od = staging_tensors(eng, 40)
    qd.copy_(torch.from_numpy(q.view(np.int16)))
    torch.cuda.synchronize()  # the engine runs on its own stream
    eng.run_device(None, 40, None)
    dst = torch.zeros((2, eng.nmod - 3, 40, 300), dtype=torch.int16, device="cuda")
    eng.rescale(40, dst, 3, True)
    torch.cuda.synchronize()
    out = od.cpu().numpy().view(np.uint16)
    got = dst.cpu().numpy().view(np.uint16)
    for part in range(2):
        cols = out[part][:, :3, :].reshape(eng.nmod, -1)  # 3 columns x 300 rows
        want = ol.rescale_oracle(cols, eng.moduli, 3, True)
        assert (got[part][:, :3, :].reshape(eng.nmod - 3, -1) == want).all()


@pytest.mark.slow
def test_ccmm_linearity_full_slice_every_element():
    # Size-independent property at the c3 slice geometry (2 parts x 2^14 rows,
    # K = 24576, N = 992): CCMM(db, q1 + q2) == CCMM(db, q1) + CCMM(db, q2)
    # mod p^2 for every one of the 2 x 24 x 992 x 2^14 outputs (the oracle
    # checks sampled rows; linearity covers the rest on the device).
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query
    N = 992
    eng = CcmmEngine(parts=2, m=1 << 14, k=24576, max_n=N)
    eng.synth_db(seed=1)
    q1 = synth_query(2, eng.K, N, eng.moduli)
    q2 = synth_query(3, eng.K, N, eng.moduli)
    mods = torch.tensor(eng.moduli, dtype=torch.int32, device="cuda").view(-1, 1, 1)
    qd, od = staging_tensors(eng, N)
    outs = []
    t1 = torch.from_numpy(q1.astype(np.int32)).cuda()
    t2 = torch.from_numpy(q2.astype(np.int32)).cuda()
    for q in (t1, t2, (t1 + t2) % mods):
        qd.copy_(q.to(torch.int16))
        torch.cuda.synchronize()  # the engine runs on its own stream
        eng.run_device(None, N, None)
        torch.cuda.synchronize()
        outs.append(od.to(torch.int32) & 0xFFFF)
    m4 = mods.view(1, -1, 1, 1)
    assert torch.equal((outs[0] + outs[1]) % m4, outs[2])
    assert bool((outs[2] < m4).all())


def test_ccmm_fused_exchange_mirrors():
    # The fused a-part exchange: the PPMM epilogue of the mirrored part stores
    # every tile locally and into each mirror buffer (peer receive buffers on a
    # multi-GPU node; same-process buffers here), for device runs and the
    # modulus-chunked e2e run alike.
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query
    n = 96
    eng = CcmmEngine(parts=2, m=520, k=640, max_n=n)
    eng.synth_db(seed=4)
    qd, od = staging_tensors(eng, n)
    mirrors = [torch.full((eng.nmod, n, 520), 7, dtype=torch.int16, device="cuda") for _ in range(2)]
    eng.set_mirror_ptrs(1, n, mirrors)
    q = synth_query(5, eng.K, n, eng.moduli)
    qd.copy_(torch.from_numpy(q.view(np.int16)))
    torch.cuda.synchronize()  # the engine runs on its own stream
    eng.run_device(None, n, None)
    torch.cuda.synchronize()
    for mbuf in mirrors:
        assert torch.equal(mbuf, od[1])
    # e2e (modulus chunks: mirror offsets follow the chunk)
    q2 = synth_query(6, eng.K, n, eng.moduli)
    out = eng.run(q2)
    torch.cuda.synchronize()
    for mbuf in mirrors:
        assert (mbuf.cpu().numpy().view(np.uint16) == out[1]).all()
    # the double-buffered receive buffer of an engine: slot 0, then slot 1
    # while slot 0 keeps the previous step, and disabling
    view, handle = eng.alloc_recv(n)
    assert len(handle) == 64 and tuple(view.shape) == (2, eng.nmod, n, 520)
    eng.set_mirror_ptrs(0, n, [view])
    eng.run_device(None, n, None)
    torch.cuda.synchronize()
    assert torch.equal(view[0], od[0])
    step0 = view[0].clone()
    eng.set_mirror_slot(1)
    qd.copy_(torch.from_numpy(q.view(np.int16)))  # staging held q2 (the e2e run above)
    torch.cuda.synchronize()
    eng.run_device(None, n, None)
    torch.cuda.synchronize()
    assert torch.equal(view[1], od[0]) and torch.equal(view[0], step0) and not torch.equal(view[0], view[1])
    with pytest.raises(Exception):
        eng.set_mirror_slot(2)
    eng.set_mirror_slot(0)
    eng.set_mirror_ptrs(0, n, [])
    before = view.clone()
    qd.copy_(torch.from_numpy(q.view(np.int16)))
    torch.cuda.synchronize()
    eng.run_device(None, n, None)
    torch.cuda.synchronize()
    assert torch.equal(view, before)


def test_blocking_api_is_thread_safe_per_context(mm):
    # the free functions are pure and reentrant; the C ABI
    # serialises calls on one context with its mutex, so concurrent host
    # threads get exact, independent results
    import threading
    p = 149
    rng = np.random.default_rng(11)
    cases = [(rng.integers(0, p * p, (40, 300)), rng.integers(0, p * p, (300, 50))) for _ in range(6)]
    want = [mm.gemm_mod_psq(a, b, p) for a, b in cases]
    got = [None] * len(cases)
    errors = []

    def work(i):
        try:
            for _ in range(5):
                got[i] = mm.gemm_mod_psq(cases[i][0], cases[i][1], p)
        except Exception as ex:  # noqa: BLE001
            errors.append(ex)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors
    for w, g in zip(want, got):
        assert (w == g).all()


def test_ccmm_run_dq_equals_run():
    # device-resident query, host outputs (the sharded-H2D multi-GPU e2e path)
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query
    eng = CcmmEngine(parts=3, m=520, k=700, max_n=96)
    eng.synth_db(seed=8)
    q = synth_query(9, eng.K, 96, eng.moduli)
    want = eng.run(q)
    qd, _ = staging_tensors(eng, 96)
    qd.copy_(torch.from_numpy(q.view(np.int16)))
    out = np.zeros_like(want)
    eng.run_dq(None, 96, out)  # ordered after the copy on torch's current stream
    assert (out == want).all()
    dq = torch.from_numpy(q.view(np.int16)).cuda()
    out2 = np.zeros_like(want)
    eng.run_dq(dq, 96, out2)
    assert (out2 == want).all()


@pytest.mark.parametrize("n", [1100, 1024, 2000])
def test_ccmm_cluster_path_padded_n_chunks(n):
    # >= 256 units so the 1x4 multicast clusters run (not the short-launch
    # plain pairs); N not a multiple of the 1024-column n-chunk -> a padded
    # last chunk whose empty tiles store nothing
    from paper_2601_17561_b200.ccmm import CcmmEngine, synth_query
    from paper_2601_17561_b200.modmat import Modulus, RnsBasis, build_paper_basis
    full = build_paper_basis()
    b = RnsBasis()
    for md in full.moduli[:4]:
        b.moduli.append(Modulus(md.p, md.e))
        b.Q *= md.p ** md.e
    eng = CcmmEngine(parts=1, m=1 << 14, k=512, max_n=n, basis=b)  # 64 m-blocks x 4 primes = 256 units
    eng.synth_db(seed=12)
    q = synth_query(13, eng.K, n, eng.moduli)
    import torch
    from paper_2601_17561_b200.ccmm import staging_tensors
    qd, od = staging_tensors(eng, n)
    qd.copy_(torch.from_numpy(q.view(np.int16)))
    eng.run_device(None, n, None)  # one launch over all 4 primes (the e2e path chunks by modulus)
    torch.cuda.synchronize()
    out = od.cpu().numpy().view(np.uint16)
    _check_ccmm(eng, 12, q, out, np.array([0, 255, 256, 9000, 16383], np.uint32))


def test_ccmm_load_part_file_streams_reference_format(tmp_path):
    # f3: the reference's BigMatrix file (save_big_matrix, modmat.cpp:216-231)
    # streamed into a part equals load_part_bigint of the same entries; header
    # and truncation errors as load_big_matrix
    from paper_2601_17561_b200.ccmm import CcmmEngine, synth_query
    from paper_2601_17561_b200.modmat import Error, ShapeMismatch
    m, k, n = 300, 640, 40
    eng = CcmmEngine(parts=2, m=m, k=k, max_n=n)
    Q = eng.basis.Q
    width = (Q.bit_length() + 7) // 8
    rng = np.random.default_rng(21)
    ent = rng.integers(0, 256, (m * k, width), dtype=np.uint8)
    ent[:, -1] = 0                          # every entry below 2^360 < Q (Q has 361 bits)
    assert 1 << (8 * (width - 1)) < Q
    path = tmp_path / "part.bin"
    with open(path, "wb") as f:
        f.write(f"{m} {k} {Q}\n".encode())
        f.write(ent.tobytes())
    eng.load_part_file(0, path)
    eng.load_part_bigint(1, ent.reshape(m, k, width), width)
    q = synth_query(3, k, n, eng.moduli)
    out = eng.run(q)
    assert (out[0] == out[1]).all()
    bad = tmp_path / "short.bin"
    bad.write_bytes(f"{m} {k} {Q}\n".encode() + ent.tobytes()[:1000])
    with pytest.raises(Error, match="truncated matrix file"):
        eng.load_part_file(0, bad)
    wrong = tmp_path / "dims.bin"
    wrong.write_bytes(f"{m + 1} {k} {Q}\n".encode())
    with pytest.raises(ShapeMismatch):
        eng.load_part_file(0, wrong)
    with pytest.raises(Error, match="cannot open"):
        eng.load_part_file(0, tmp_path / "missing.bin")


@pytest.mark.parametrize("devices,parts,m", [([0, 0], 3, 384), ([0, 0, 0], 3, 384), ([0, 0, 0, 0], 8, 384),
                                             ([0, 0], 4, 2560)])
def test_ccmm_group_full_equals_one_engine_and_exchanges_the_a_part(devices, parts, m):
    """irl_ccmm_full (single-process multi-GPU; here every rank on device 0):
    the parts dealt as dist.part_range, every rank's outputs in global order,
    equal to one engine holding all parts; every rank ends with the a-part
    result, stored into it by rank 0's PPMM epilogue (fused exchange)."""
    import torch

    from paper_2601_17561_b200 import capi
    from paper_2601_17561_b200.ccmm import CcmmEngine, CcmmGroup, synth_query
    from paper_2601_17561_b200.dist import part_range
    # m = 2560: 10 row blocks x 2 parts x 24 moduli = 480 units per rank, so
    # every rank's launch plans the 1x4-cluster grid plus its filler grid,
    # concurrently on one device from two host threads
    k, n = 1024, 96
    g = CcmmGroup(devices, parts=parts, m=m, k=k, max_n=n)
    try:
        for r in range(len(devices)):
            _, first, count = g.engine(r)
            pr = part_range(r, len(devices), parts)
            assert (first, count) == (pr.first, pr.count)
        g.synth_db(seed=1)
        eng = CcmmEngine(parts=parts, m=m, k=k, max_n=n)
        eng.synth_db(seed=1)
        q = synth_query(2, k, n, eng.moduli)
        want = eng.run(q)
        q2 = synth_query(3, k, n, eng.moduli)
        want2 = eng.run(q2)
        eng.close()
        out, ptrs, mode = g.run(q)
        assert mode == capi.IRL_EXCHANGE_P2P  # ranks share a device: no multicast, P2P stores
        assert np.array_equal(out, want)
        torch.cuda.synchronize()
        for r in range(len(devices)):
            a = g.a_part(r, ptrs[r], n).cpu().numpy().view(np.uint16)
            assert np.array_equal(a, want[0]), r
        # a second call reuses the exchange set-up and stores the a-part into
        # the other receive slot: the first call's copy stays intact
        out2, ptrs2, _ = g.run(q2)
        assert np.array_equal(out2, want2)
        torch.cuda.synchronize()
        for r in range(1, len(devices)):
            assert ptrs2[r] != ptrs[r]
            assert np.array_equal(g.a_part(r, ptrs2[r], n).cpu().numpy().view(np.uint16), want2[0]), r
            assert np.array_equal(g.a_part(r, ptrs[r], n).cpu().numpy().view(np.uint16), want[0]), r
        out3, ptrs3, _ = g.run(q)  # third call: back to the first slot
        assert np.array_equal(out3, want) and ptrs3[-1] == ptrs[-1]
        # the sharded query distribution (each rank's moduli from the host, then
        # a peer all-gather, then irl_ccmm_run_dq) and the whole-query copies
        # give the same outputs and the same a-part on every rank
        for shard in (1, 0, -1):
            g.set_query_shard(shard)
            outs, ptrs_s, mode_s = g.run(q2)
            assert mode_s == capi.IRL_EXCHANGE_P2P and np.array_equal(outs, want2), shard
            torch.cuda.synchronize()
            for r in range(len(devices)):
                assert np.array_equal(g.a_part(r, ptrs_s[r], n).cpu().numpy().view(np.uint16), want2[0]), (shard, r)
    finally:
        g.close()


def test_ccmm_group_rejects_more_devices_than_parts():
    from paper_2601_17561_b200.ccmm import CcmmGroup
    from paper_2601_17561_b200.modmat import ShapeMismatch
    with pytest.raises(ShapeMismatch):
        CcmmGroup([0, 0, 0], parts=2, m=128, k=256, max_n=32)


@pytest.mark.parametrize("k", [1024, 4096])
def test_ccmm_group_nvls_multicast_mirror(k):
    """The NVLS multicast exchange on one GPU: a multicast object with this
    device, the rank's receive buffer bound to it, and the a-part PPMM epilogue
    storing every pair of output rows once through the multicast address
    (multimem.st). With one device the switch delivers to that one copy; on an
    NVSwitch node the same stores reach every rank. k = 4096 exercises the
    K-chunked (accumulating) launches when the digit bound requires them."""
    import torch

    from paper_2601_17561_b200 import capi
    from paper_2601_17561_b200.ccmm import CcmmEngine, CcmmGroup, synth_query
    m, n = 384, 96
    g = CcmmGroup([0], parts=2, m=m, k=k, max_n=n)
    from paper_2601_17561_b200.modmat import Error
    try:
        g.synth_db(seed=4)
        g.set_exchange(capi.IRL_EXCHANGE_MULTICAST)
        eng = CcmmEngine(parts=2, m=m, k=k, max_n=n)
        eng.synth_db(seed=4)
        q = synth_query(5, k, n, eng.moduli)
        want = eng.run(q)
        eng.close()
        try:
            out, ptrs, mode = g.run(q)
        except Error as ex:  # containers without the NVSwitch fabric refuse cuMulticastCreate
            if "multicast" in str(ex):
                pytest.skip(f"NVLS multicast unavailable here: {ex}")
            raise
        assert mode == capi.IRL_EXCHANGE_MULTICAST
        assert np.array_equal(out, want)
        torch.cuda.synchronize()
        a = g.a_part(0, ptrs[0], n).cpu().numpy().view(np.uint16)
        assert np.array_equal(a, want[0])
        # the multicast copy is rewritten on every run, and a narrower batch re-binds
        q2 = synth_query(6, k, n, eng.moduli)
        out2, ptrs2, _ = g.run(q2)
        torch.cuda.synchronize()
        assert np.array_equal(g.a_part(0, ptrs2[0], n).cpu().numpy().view(np.uint16), out2[0])
        q3 = np.ascontiguousarray(q2[:, :, :64])
        out3, ptrs3, mode3 = g.run(q3)
        torch.cuda.synchronize()
        assert mode3 == capi.IRL_EXCHANGE_MULTICAST
        assert np.array_equal(g.a_part(0, ptrs3[0], 64).cpu().numpy().view(np.uint16), out3[0])
    finally:
        g.close()


def test_ccmm_row_blocks_synth_and_multi_part_mirror():
    """Row-block units (dist.deal_blocks): synth_part fills a unit with rows
    [row0, row0 + M) of a taller global part, identical to the same rows of a
    whole-part engine; a mirror spanning several units (an a-part dealt as
    blocks) lands back to back in the peer buffer, in the double-buffered slot."""
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query
    k, n, blk = 640, 64, 256
    whole = CcmmEngine(parts=2, m=4 * blk, k=k, max_n=n)
    whole.synth_db(seed=6)
    q = synth_query(7, k, n, whole.moduli)
    want = whole.run(q)                      # [2][nmod][n][1024]
    whole.close()
    units = [(0, 0), (0, 256), (0, 512), (1, 768), (1, 0)]
    eng = CcmmEngine(parts=len(units), m=blk, k=k, max_n=n)
    for j, (gp, r0) in enumerate(units):
        eng.synth_part(j, 6, gp, r0)
    view, _ = eng.alloc_recv(n, parts=3)
    assert tuple(view.shape) == (2, 3, eng.nmod, n, blk)
    eng.set_mirror_ptrs(0, n, [view])
    eng.set_mirror_parts(3)
    eng.set_mirror_slot(1)
    got = eng.run(q)
    torch.cuda.synchronize()
    for j, (gp, r0) in enumerate(units):
        assert np.array_equal(got[j], want[gp][:, :, r0:r0 + blk]), j
    mv = view.cpu().numpy().view(np.uint16)
    assert np.array_equal(mv[1], got[:3]) and not mv[0].any()
    with pytest.raises(Exception):
        eng.set_mirror_parts(6)


def test_ccmm_run_pageable_and_pinned_buffers_agree():
    """irl_ccmm_run stages pageable caller buffers in page-locked memory (query
    up front, each D2H block copied out as it lands); page-locked buffers are
    DMA'd directly. Both give the same outputs, and the pinned output buffer
    is written in place."""
    import torch

    from paper_2601_17561_b200.ccmm import CcmmEngine, synth_query
    eng = CcmmEngine(parts=3, m=640, k=1536, max_n=160)
    eng.synth_db(seed=9)
    q = synth_query(10, eng.K, 160, eng.moduli)
    out_pageable = eng.run(q)
    qp = torch.from_numpy(q.view(np.int16)).pin_memory().numpy().view(np.uint16)
    op = torch.zeros(out_pageable.shape, dtype=torch.int16).pin_memory().numpy().view(np.uint16)
    out_pinned = eng.run(qp, op)
    assert out_pinned is op and np.array_equal(out_pinned, out_pageable)
    again = eng.run(q)  # the staging buffers are reused
    assert np.array_equal(again, out_pageable)
    _check_ccmm(eng, 9, q, out_pageable, np.array([0, 333, 639], np.uint32))
    eng.close()


@pytest.mark.parametrize("m,k,n", [(0, 5, 3), (2, 0, 3), (2, 3, 0), (1, 1, 1)])
def test_gemm_mod_Q_empty_and_unit_shapes(mm, basis, m, k, n):
    """gemm_mod_Q (modmat.cpp:162-195) on empty and 1x1x1 shapes: same shape
    and entries as the oracle (an empty inner dimension gives zeros mod Q)."""
    rng = np.random.default_rng(m * 100 + k * 10 + n)
    Q = basis.Q
    a = mm.BigMatrix(m, k, [int(rng.integers(0, 1 << 62)) * int(rng.integers(1, 1 << 62)) % Q for _ in range(m * k)])
    b = mm.BigMatrix(k, n, [int(rng.integers(0, 1 << 62)) * int(rng.integers(1, 1 << 62)) % Q for _ in range(k * n)])
    c = mm.gemm_mod_Q(a, b, basis)
    assert (c.rows, c.cols) == (m, n)
    want = [sum(a.a[i * k + t] * b.a[t * n + j] for t in range(k)) % Q for i in range(m) for j in range(n)]
    assert c.a == want

"""f1: the B200 CCMM under the reference's own caller. Emulator::ccmm_twin
(emulator.cpp:389-447) is the CCMM call site of run_alg1 / run_alg2
(pipeline.cpp:512-514, 550-557). Two libraries are built from the unmodified
reference sources (oracle/Makefile `pipe`): stock, and with ccmm_twin's product
from the B200 engine (paper_2601_17561_b200/host/emulator_ccmm_hook.cpp,
interposed with -Wl,--wrap). The reference's own end-to-end scenarios
(test_pipeline.cpp:254-299; acceptance.cpp:187-312 criteria 6 and 7) must give
identical match bits, oracle agreement, bootstrap counts, trace lengths and a
bit-identical digest of every ccmm_twin output message.

Also: irl_ccmm_twin on arbitrary doubles (the FP64 path) against the oracle
restatement of the reference loop, bit for bit."""
import numpy as np
import pytest

import oracle_lib as ol

pytestmark = pytest.mark.gpu

needs_pipe = pytest.mark.skipif(not ol.pipe_available(), reason="oracle/_ref pipe libraries not built")


def _spec(**kw):
    from paper_2601_17561_b200.ccmm import CcmmSpec
    base = dict(d1=4, d2=3, d3=2, n_db=2, n_qry=3, db_modulus_bits=40.0, qry_modulus_bits=30.0, scale_bits=20.0)
    base.update(kw)
    return CcmmSpec(**base)


@pytest.mark.parametrize("d1,d2,d3,n_db,seed", [(64, 48, 6, 16, 1), (1024, 512, 70, 256, 2), (96, 1000, 33, 32, 3)])
def test_ccmm_twin_arbitrary_doubles_bitexact(d1, d2, d3, n_db, seed):
    """Non-integer messages: the ordered FP64 kernel replays the reference's
    rounded multiply / add per k, zero database entries skipped, inf and NaN
    propagated -- identical bit patterns to the oracle restatement (itself
    pinned to the reference in tests/test_oracle.py)."""
    from paper_2601_17561_b200.ccmm import ccmm_twin
    db, qry = ol.twin_doubles(d1, d2, d3, seed)
    qry[min(3, d2 - 1), min(2, d3 - 1)] = np.inf
    db[0, 0], qry[0, min(4, d3 - 1)] = np.inf, 0.0
    out = ccmm_twin(_spec(d1=d1, d2=d2, d3=d3, n_db=n_db, n_qry=d2), db, qry, top_level=9)
    want = ol.orc_ccmm_twin_product(db, qry).reshape(-1, n_db)
    assert np.array_equal(out.messages.view(np.uint64), want.view(np.uint64))


def test_ccmm_twin_large_integers_take_the_fp64_path():
    # integers whose partial sums pass 2^52: the reference's double rounding
    # is reproduced instead of the exact product
    from paper_2601_17561_b200.ccmm import ccmm_twin
    rng = np.random.default_rng(4)
    d1, d2, d3 = 128, 64, 8
    db = rng.integers(-(1 << 30), 1 << 30, (d1, d2)).astype(np.float64)
    qry = rng.integers(-(1 << 30), 1 << 30, (d2, d3)).astype(np.float64)
    out = ccmm_twin(_spec(d1=d1, d2=d2, d3=d3, n_db=32, n_qry=d2), db, qry, top_level=9)
    want = ol.orc_ccmm_twin_product(db, qry).reshape(-1, 32)
    assert np.array_equal(out.messages.view(np.uint64), want.view(np.uint64))


@pytest.mark.skipif(not ol.ref_available(), reason="oracle/_ref not built")
def test_ccmm_twin_matches_reference_emulator_directly():
    # the reference's own Emulator::ccmm_twin (oracle/_ref) vs irl_ccmm_twin:
    # integer (tensor-core) and fractional (FP64) operands
    from paper_2601_17561_b200.ccmm import ccmm_twin
    rng = np.random.default_rng(8)
    for db, qry in [(rng.integers(-1, 2, (256, 128)).astype(np.float64), rng.integers(-1, 2, (128, 31)).astype(np.float64)),
                    ol.twin_doubles(256, 128, 31, 9)]:
        st, want, top = ol.ref_ccmm_twin(db, qry, 64, 128)
        assert st == 0
        out = ccmm_twin(_spec(d1=256, d2=128, d3=31, n_db=64, n_qry=128, db_modulus_bits=100.0,
                              qry_modulus_bits=50.0, scale_bits=23.0), db, qry, top_level=top)
        assert np.array_equal(out.messages.ravel().view(np.uint64), want.ravel().view(np.uint64))


def _run_planted(kind):
    lib = ol.pipe(kind)
    lib.irl_hook_reset()
    out = np.zeros(64, np.int64)
    st = lib.pipe_planted_small(ol.ptr(out, ol.i64p))
    assert st == 0, lib.pipe_last_error()
    return out, lib.irl_hook_digest(), lib.irl_hook_calls(), lib.irl_hook_slots(), lib.irl_hook_is_b200()


@needs_pipe
def test_reference_pipeline_planted_match_through_b200():
    """test_pipeline.cpp:254-299 with the B200 product underneath run_alg1 and
    run_alg2: the reference's assertions hold, and every result equals the
    stock reference's."""
    stock, d_s, calls_s, slots_s, is_b_s = _run_planted("ref")
    b200, d_b, calls_b, slots_b, is_b_b = _run_planted("b200")
    assert (is_b_s, is_b_b) == (0, 1)
    r1, r2, r3 = b200[:16], b200[16:32], b200[32:48]
    assert b200[48] == 1                       # the planted score lies in P
    assert r1[7] == 1 and r1[8] == 1 and r1[0] == 1   # alg1: match bit 1, oracle 1, agrees
    assert r1[2] == 8                          # bts_pre == rho
    assert r2[0] == 1 and r2[1] == 1 and r2[2] == 2   # alg2 agrees, folding ok, ceil(rho/k)
    assert r1[2] == 4 * r2[2]                  # k | rho: exactly k times fewer
    assert r3[7] == 0 and r3[8] == 0 and r3[0] == 1   # clean query stays negative
    assert (b200 == stock).all()
    assert calls_b == calls_s == 3 and slots_b == slots_s > 0
    assert d_b == d_s                          # every ccmm_twin message bit-identical


@needs_pipe
@pytest.mark.parametrize("rho,batch,n_db,instances,seed0", [(31, 4, 4096, 2, 60000), (32, 1, 1024, 1, 70000)])
def test_acceptance_criteria_6_7_through_b200(rho, batch, n_db, instances, seed0):
    """acceptance.cpp:187-312 run_instances() on full_config (n_db 4096, d 1024,
    rho 31, batch 4, planted matches) and criterion 7's rho = 32 run, with the
    B200 product: oracle agreement, folding assumption, bootstrap accounting
    (alg1 = k * alg2 at k | rho), all equal to the stock reference."""
    fc = np.ascontiguousarray(ol.FOLD_POLY_APPC, np.float64)
    res, dig = {}, {}
    for kind in ("ref", "b200"):
        lib = ol.pipe(kind)
        lib.irl_hook_reset()
        stride = 7 + 2 * batch
        out = np.zeros((instances, 2, stride), np.int64)
        st = lib.pipe_instances(rho, batch, n_db, instances, seed0, fc.ctypes.data_as(ol.C.POINTER(ol.C.c_double)),
                                len(fc), ol.ptr(out, ol.i64p), stride)
        assert st == 0, lib.pipe_last_error()
        res[kind], dig[kind] = out, (lib.irl_hook_digest(), lib.irl_hook_calls(), lib.irl_hook_slots())
    out = res["b200"]
    assert (out == res["ref"]).all()
    assert dig["b200"] == dig["ref"] and dig["b200"][1] == 2 * instances
    for inst in range(instances):
        a1, a2 = out[inst, 0], out[inst, 1]
        assert a1[0] == 1 and a2[0] == 1          # both agree with the plaintext oracle
        assert (a1[7:7 + batch] == a2[7:7 + batch]).all()
        assert a2[1] == 1                         # folding assumption held
        k = 16
        if rho % k == 0:
            assert a1[2] == k * a2[2]
        else:
            assert 0 <= k * a2[2] - a1[2] <= (k - 1) * (n_db // 1024) * batch


@needs_pipe
@pytest.mark.slow
def test_acceptance_criteria_6_7_in_full_through_b200():
    """acceptance.cpp:268-312 criteria 6 and 7 exactly as the reference states
    them, with every CCMM product from the B200: 100 full_config instances from
    seed 60000 all agree with the plaintext oracle with the folding assumption
    held; pre-classification bootstraps alg1 = k * alg2 up to the ceiling slack
    (k - 1) per (block, eye); total ratio >= k; the rho = 32 run exactly k."""
    fc = np.ascontiguousarray(ol.FOLD_POLY_APPC, np.float64)
    lib = ol.pipe("b200")
    f64p = ol.C.POINTER(ol.C.c_double)

    def run(rho, batch, n_db, instances, seed0):
        stride = 7 + 2 * batch
        out = np.zeros((instances, 2, stride), np.int64)
        st = lib.pipe_instances(rho, batch, n_db, instances, seed0, fc.ctypes.data_as(f64p), len(fc),
                                ol.ptr(out, ol.i64p), stride)
        assert st == 0, lib.pipe_last_error()
        return out

    k, batch, n_db, d = 16, 4, 4096, 1024
    out = run(31, batch, n_db, 100, 60000)
    a1, a2 = out[:, 0], out[:, 1]
    # criterion 6: r1, r2 agree with the oracle and with each other; folding ok
    assert (a1[:, 0] == 1).all() and (a2[:, 0] == 1).all() and (a2[:, 1] == 1).all()
    assert (a1[:, 7:7 + batch] == a2[:, 7:7 + batch]).all()
    assert a1[:, 7:7 + batch].any()          # planted matches were found
    # criterion 7: bootstrap accounting
    alg1_pre, alg2_pre = int(a1[:, 2].sum()), int(a2[:, 2].sum())
    b_units = (n_db // d) * batch * 100
    deficit = k * alg2_pre - alg1_pre
    assert 0 <= deficit <= (k - 1) * b_units
    total1 = int(a1[:, 2:5].sum())
    total2 = int(a2[:, 2:5].sum())
    assert total1 / max(1, total2) >= k
    ex = run(32, 1, 1024, 1, 70000)
    assert ex[0, 1, 2] > 0 and ex[0, 0, 2] == k * ex[0, 1, 2]
    # the first instances equal the stock reference's, message digest included
    ref = ol.pipe("ref")
    for libx in (lib, ref):
        libx.irl_hook_reset()
    head_b = run(31, batch, n_db, 3, 60000)
    stride = 7 + 2 * batch
    head_r = np.zeros_like(head_b)
    assert ref.pipe_instances(31, batch, n_db, 3, 60000, fc.ctypes.data_as(f64p), len(fc),
                              ol.ptr(head_r, ol.i64p), stride) == 0
    assert (head_b == head_r).all() and (head_b == out[:3]).all()
    assert lib.irl_hook_digest() == ref.irl_hook_digest()

"""Alg. 2 fold stage (reference pipeline.cpp:359-408, 538-633).

CPU: the oracle restatement (oracle/irl_oracle.c orc_fold_stage) against the
golden vectors the reference itself produced (tests/golden/fold_stage.npz:
pipe::normalize / fold_group / eval_chain_ct on a noise-free emulator, and
run_alg2's folding-assumption flag), and against oracle/_ref on fresh random
inputs when it was built here.

GPU: csrc/fold.cu through the C ABI (irl_fold_stage, irl_fold_stage_device,
irl_iris_db_fold) against the same golden vectors and the oracle, bit for
bit (IEEE double, no contraction), plus the reference's error behaviour.
"""
import numpy as np
import pytest

import oracle_lib as ol

GOLD = np.load(ol.ROOT / "tests" / "golden" / "fold_stage.npz")
CASES = ["dense", "wide", "single", "ragged", "zero"]
ref_only = pytest.mark.skipif(not ol.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


def case(tag):
    d, blocks, batch, rho, fold_k = (int(v) for v in GOLD[f"{tag}_params"])
    return dict(d=d, blocks=blocks, batch=batch, rho=rho, fold_k=fold_k,
                neg=tuple(GOLD[f"{tag}_negative"]), chain=ol.fold_chain_for_tests(str(GOLD[f"{tag}_chain"])),
                inner=GOLD[f"{tag}_inner"], overlap=GOLD[f"{tag}_overlap"], status=int(GOLD[f"{tag}_status"]),
                folded=GOLD[f"{tag}_folded"], refolded=GOLD[f"{tag}_refolded"],
                ok=int(GOLD[f"{tag}_assumption_ok"]))


# ---------------------------------------------------------------- CPU oracle

@pytest.mark.parametrize("tag", CASES)
def test_oracle_fold_matches_reference_golden(tag):
    c = case(tag)
    st, folded, refolded, ok = ol.orc_fold(c["inner"], c["overlap"], c["batch"], c["rho"], c["d"], c["fold_k"],
                                           GOLD["fold_poly"], c["chain"], c["neg"])
    assert st == c["status"]
    if st == 0:  # the reference stops at the first ZeroOverlap; nothing to compare
        assert np.array_equal(folded, c["folded"])
        assert np.array_equal(refolded, c["refolded"])
        assert ok == c["ok"]


def test_golden_covers_both_assumption_outcomes():
    flags = {case(t)["ok"] for t in CASES}
    assert {0, 1} <= flags


def test_oracle_config_errors_follow_validate():
    inner = np.zeros((4, 64), np.int32)
    ovl = np.ones((4, 64), np.int32)
    chain = ol.fold_chain_for_tests()
    f = ol.FOLD_POLY_APPC
    # rho / batch, fold_k, d power of two, n_db multiple of d (pipeline.cpp:233-243)
    assert ol.orc_fold(inner, ovl, 4, 0, 64, 1, f, chain, (-1, 1))[0] == 13
    assert ol.orc_fold(inner, ovl, 2, 2, 64, 3, f, chain, (-1, 1))[0] == 13
    assert ol.orc_fold(inner, ovl, 2, 2, 48, 1, f, chain, (-1, 1))[0] == 13
    assert ol.orc_fold(inner[:, :48], ovl[:, :48], 2, 2, 32, 1, f, chain, (-1, 1))[0] == 13
    assert ol.orc_fold(inner, ovl, 2, 2, 64, 1, f, [], (-1, 1))[0] == 13  # empty chain
    assert ol.orc_fold(inner, ovl, 2, 2, 64, 1, f, [], (-1, 1), want_refold=False)[0] == 0


@ref_only
@pytest.mark.parametrize("deg", list(range(0, 32)))
def test_oracle_ps_execute_equals_reference(deg):
    import ctypes as C
    rng = np.random.default_rng(deg)
    c = rng.normal(size=deg + 1) / np.arange(1, deg + 2)
    f64p = C.POINTER(C.c_double)
    for x in rng.uniform(-1.3, 1.3, size=16):
        r = C.c_double()
        assert ol.ref().ref_ps_execute(ol.ptr(c, f64p), deg + 1, x, C.byref(r)) == 0
        assert ol.oracle().orc_ps_execute(ol.ptr(c, f64p), deg + 1, x) == r.value


@ref_only
@pytest.mark.parametrize("seed,kind", [(1, "step"), (2, "wide"), (3, "random")])
def test_oracle_fold_equals_reference_random(seed, kind):
    rng = np.random.default_rng(seed)
    d, blocks, batch, rho, fold_k = 32, 3, 2, 9, 4
    n_db = d * blocks
    ovl = rng.integers(1, 300, size=(batch * rho, n_db)).astype(np.int32)
    inner = (rng.integers(-300, 301, size=ovl.shape) % (ovl + 1)).astype(np.int32)
    inner *= np.where(rng.random(ovl.shape) < 0.5, -1, 1).astype(np.int32)
    if kind == "random":
        fold_c = rng.normal(size=12) / np.arange(1, 13) ** 2
        chain = [(0.1, rng.normal(size=6) / 4), (-0.2, rng.normal(size=17) / np.arange(1, 18) ** 2)]
    else:
        fold_c, chain = ol.FOLD_POLY_APPC, ol.fold_chain_for_tests(kind)
    st_r, f_r, r_r = ol.ref_fold(inner, ovl, batch, rho, d, fold_k, fold_c, chain)
    st_o, f_o, r_o, _ = ol.orc_fold(inner, ovl, batch, rho, d, fold_k, fold_c, chain, (-0.25, 0.25))
    assert st_r == st_o == 0
    assert np.array_equal(f_o, f_r, equal_nan=True) and np.array_equal(r_o, r_r, equal_nan=True)


@ref_only
def test_oracle_assumption_flag_equals_reference_run_alg2():
    for k, (d, blocks, batch, rho, fold_k, neg) in enumerate(
            [(64, 2, 2, 6, 2, (-0.25, 0.25)), (64, 2, 2, 6, 6, (-0.35, 0.35)), (32, 4, 1, 7, 3, (-1.0, 1.0))]):
        dc, dm = ol.ref_synth_templates(d * blocks, d, 0.8, 100 + k)
        qc, qm = ol.ref_synth_templates(batch, d, 0.8, 200 + k)
        inner, ovl = ol.orc_inner_overlap(dc, dm, qc, qm, rho)
        chain = ol.fold_chain_for_tests()
        _, _, _, ok = ol.orc_fold(inner, ovl, batch, rho, d, fold_k, ol.FOLD_POLY_APPC, chain, neg)
        assert ok == ol.ref_alg2_flag(qc, qm, dc, dm, rho, fold_k, ol.FOLD_POLY_APPC, chain, neg)


# ---------------------------------------------------------------- GPU

def _cfg(c, fold_poly=None, chain=None):
    from paper_2601_17561_b200.fold import FoldConfig
    return FoldConfig(rho=c["rho"], fold_k=c["fold_k"], d=c["d"],
                      fold_poly=GOLD["fold_poly"] if fold_poly is None else fold_poly,
                      fold_chain=c["chain"] if chain is None else chain, negative=c["neg"])


@pytest.mark.gpu
@pytest.mark.parametrize("tag", CASES)
def test_gpu_fold_stage_golden(tag):
    from paper_2601_17561_b200.fold import fold_stage
    from paper_2601_17561_b200.modmat import ZeroOverlap
    c = case(tag)
    if c["status"] == 11:
        with pytest.raises(ZeroOverlap):
            fold_stage(c["inner"], c["overlap"], c["batch"], _cfg(c))
        return
    res = fold_stage(c["inner"], c["overlap"], c["batch"], _cfg(c))
    assert np.array_equal(res.folded.ravel(), c["folded"])
    assert np.array_equal(res.refolded.ravel(), c["refolded"])
    assert int(res.assumption_ok) == c["ok"]


@pytest.mark.gpu
@pytest.mark.parametrize("tag", CASES)
def test_gpu_iris_db_fold_from_templates_golden(tag):
    """The whole post-CCMM path from templates: int8-GEMM products and overlaps
    on the device, then the fold stage; equals the reference's messages."""
    from paper_2601_17561_b200.iris import IrisDatabase, pack_bits
    from paper_2601_17561_b200.modmat import ZeroOverlap
    c = case(tag)
    dc, dm = GOLD[f"{tag}_db_code"], GOLD[f"{tag}_db_mask"]
    qc, qm = GOLD[f"{tag}_q_code"], GOLD[f"{tag}_q_mask"]
    db = IrisDatabase.from_packed(pack_bits(dc), pack_bits(dm), c["d"], max_cols=c["batch"] * c["rho"])
    try:
        if c["status"] == 11:
            with pytest.raises(ZeroOverlap):
                db.fold_packed(pack_bits(qc), pack_bits(qm), c["batch"], _cfg(c))
            return
        res = db.fold_packed(pack_bits(qc), pack_bits(qm), c["batch"], _cfg(c))
        assert np.array_equal(res.folded.ravel(), c["folded"])
        assert np.array_equal(res.refolded.ravel(), c["refolded"])
        assert int(res.assumption_ok) == c["ok"]
    finally:
        db.close()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_gpu_fold_every_degree_vs_oracle(seed):
    """Random polynomials of every degree 0..31 as fold polynomial and chain
    stages (the kernel's compile-time Paterson-Stockmeyer plans), ragged last
    group, several blocks; bit-exact against the oracle."""
    from paper_2601_17561_b200.fold import FoldConfig, fold_stage
    rng = np.random.default_rng(seed)
    d, blocks, batch, rho, fold_k = 256, 3, 3, 11, 4
    n_db = d * blocks
    ovl = rng.integers(1, 2000, size=(batch * rho, n_db)).astype(np.int32)
    inner = (rng.integers(-2000, 2001, size=ovl.shape) % (ovl + 1)).astype(np.int32)
    inner *= np.where(rng.random(ovl.shape) < 0.5, -1, 1).astype(np.int32)
    for deg in range(seed, 32, 3):
        fold_c = rng.normal(size=deg + 1) / np.arange(1, deg + 2) ** 2
        sd = (deg * 7 + 3) % 32
        chain = [(0.05, rng.normal(size=sd + 1) / np.arange(1, sd + 2) ** 2), (-0.1, rng.normal(size=4) / 3)]
        neg = (-0.2, 0.2)
        cfg = FoldConfig(rho=rho, fold_k=fold_k, d=d, fold_poly=fold_c, fold_chain=chain, negative=neg)
        res = fold_stage(inner, ovl, batch, cfg)
        st, f_o, r_o, ok = ol.orc_fold(inner, ovl, batch, rho, d, fold_k, fold_c, chain, neg)
        assert st == 0
        assert np.array_equal(res.folded.ravel(), f_o, equal_nan=True), deg
        assert np.array_equal(res.refolded.ravel(), r_o, equal_nan=True), deg
        assert res.assumption_ok == bool(ok)


@pytest.mark.gpu
def test_gpu_fold_stage_device_flags_and_streams():
    import torch

    from paper_2601_17561_b200.fold import fold_stage_device
    c = case("dense")
    cfg = _cfg(c)
    inner = torch.from_numpy(c["inner"]).cuda()
    ovl = torch.from_numpy(c["overlap"]).cuda()
    groups = -(-c["rho"] // c["fold_k"])
    folded = torch.empty(c["batch"] * c["blocks"] * groups * c["d"], dtype=torch.float64, device="cuda")
    refolded = torch.empty(c["batch"] * c["blocks"] * c["d"], dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        flags = fold_stage_device(inner, ovl, c["batch"], cfg, folded, refolded)
    s.synchronize()
    assert np.array_equal(folded.cpu().numpy(), c["folded"])
    assert np.array_equal(refolded.cpu().numpy(), c["refolded"])
    assert flags.cpu().tolist() == [1 - c["ok"], 0]
    # an empty overlap sets flag 1 instead of raising
    ovl[0, 3] = 0
    flags = fold_stage_device(inner, ovl, c["batch"], cfg, folded, None)
    torch.cuda.synchronize()
    assert flags.cpu().tolist()[1] == 1


@pytest.mark.gpu
def test_gpu_fold_config_errors_follow_validate():
    from paper_2601_17561_b200.fold import FoldConfig, fold_stage
    from paper_2601_17561_b200.modmat import ConfigError
    inner = np.zeros((4, 64), np.int32)
    ovl = np.ones((4, 64), np.int32)
    chain = ol.fold_chain_for_tests()
    cases = [
        (FoldConfig(rho=0, fold_k=1, d=64, fold_chain=chain), 4, "pipeline: rho and batch must be >= 1"),
        (FoldConfig(rho=2, fold_k=3, d=64, fold_chain=chain), 2, "pipeline: fold_k must satisfy 1 <= k <= rho"),
        (FoldConfig(rho=2, fold_k=1, d=48, fold_chain=chain), 2, "pipeline: d must be a power of two"),
        (FoldConfig(rho=2, fold_k=1, d=128, fold_chain=chain), 2, "pipeline: n_db must be a positive multiple of d"),
    ]
    for cfg, batch, msg in cases:
        with pytest.raises(ConfigError, match=msg):
            fold_stage(inner, ovl, batch, cfg)
    with pytest.raises(ConfigError, match="eval_chain_ct: empty chain"):
        fold_stage(inner, ovl, 2, FoldConfig(rho=2, fold_k=1, d=64), want_refolded=True)
    res = fold_stage(inner, ovl, 2, FoldConfig(rho=2, fold_k=1, d=64))  # no chain: folded only
    assert res.refolded is None and res.folded.shape == (2, 1, 2, 64)


@pytest.mark.gpu
def test_gpu_fold_paper_scale_eyes_vs_oracle():
    """Paper geometry through irl_iris_db_fold: 7 * 2^14 templates of
    d = 2^14 (blocks = 7), 32 eyes x 31 rotations, fold_k = 16. Two eyes are
    checked bit-exactly against the oracle on the GPU's own products and
    overlaps (irl_iris_inner_overlap, pinned by test_iris.py)."""
    import ctypes as C

    from paper_2601_17561_b200 import capi
    from paper_2601_17561_b200.fold import FoldConfig
    from paper_2601_17561_b200.iris import IrisDatabase
    from paper_2601_17561_b200.modmat import default_context
    rng = np.random.default_rng(5)
    d, n_db, eyes, rho, words = 1 << 14, 7 << 14, 32, 31, (1 << 14) // 64
    bits = lambda n: rng.integers(0, 1 << 63, size=(n, words), dtype=np.uint64) ^ \
        rng.integers(0, 2, size=(n, words), dtype=np.uint64) << np.uint64(63)  # noqa: E731
    dc, qc = bits(n_db), bits(eyes)
    dm, qm = bits(n_db) | bits(n_db), bits(eyes) | bits(eyes)  # masks of density 3/4
    cfg = FoldConfig(rho=rho, fold_k=16, d=d, fold_chain=ol.fold_chain_for_tests("wide"), negative=(-0.05, 0.05))
    db = IrisDatabase.from_packed(dc, dm, d, max_cols=eyes * rho)
    try:
        res = db.fold_packed(qc, qm, eyes, cfg)
    finally:
        db.close()
    assert res.folded.shape == (eyes, 7, 2, d) and res.refolded.shape == (eyes, 7, d)
    sub = 2
    inner = np.zeros((sub * rho, n_db), np.int32)
    ovl = np.zeros_like(inner)
    ctx = default_context()
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    ctx.check(capi.lib().irl_iris_inner_overlap(ctx.handle, p(dc), p(dm), n_db, p(qc), p(qm), sub, rho, d,
                                                p(inner), p(ovl)))
    st, f_o, r_o, ok = ol.orc_fold(inner, ovl, sub, rho, d, 16, cfg.fold_poly, cfg.fold_chain, cfg.negative)
    assert st == 0
    assert np.array_equal(res.folded[:sub].ravel(), f_o)
    assert np.array_equal(res.refolded[:sub].ravel(), r_o)


def _boundary_pairs():
    """(raw, ov) pairs whose quotient RN(raw/ov) differs from raw * RN(1/ov):
    one with the product below the quotient, one above."""
    below = above = None
    for ov in range(3, 200):
        for raw in range(1, 400):
            x, q = raw * (1.0 / ov), raw / ov
            if x < q and below is None:
                below = (raw, ov, q)
            if x > q and above is None:
                above = (raw, ov, q)
        if below and above:
            return below, above


@pytest.mark.gpu
@pytest.mark.parametrize("side", ["lo", "hi"])
def test_gpu_fold_shadow_check_uses_the_ieee_quotient(side):
    """The folding-assumption check compares raw / ov (IEEE quotient,
    pipeline.cpp:580) with the interval ends. Both rotations of every slot sit
    exactly on an end, where raw * RN(1/ov) would land one ulp outside: the
    reference counts them inside, so the assumption holds."""
    from paper_2601_17561_b200.fold import FoldConfig, fold_stage
    below, above = _boundary_pairs()
    raw, ov, q = below if side == "lo" else above
    neg = (q, q + 1.0) if side == "lo" else (q - 1.0, q)
    d = 2
    inner = np.full((2, d), raw, np.int32)
    ovl = np.full((2, d), ov, np.int32)
    cfg = FoldConfig(rho=2, fold_k=2, d=d, fold_chain=[], negative=neg)
    res = fold_stage(inner, ovl, 1, cfg)
    _, f_o, _, ok = ol.orc_fold(inner, ovl, 1, 2, d, 2, cfg.fold_poly, [], neg, want_refold=False)
    assert ok == 1 and res.assumption_ok
    assert np.array_equal(res.folded.ravel(), f_o)
    # one ulp further in, the pair is outside for both
    neg2 = (np.nextafter(q, np.inf), q + 1.0) if side == "lo" else (q - 1.0, np.nextafter(q, -np.inf))
    res = fold_stage(inner, ovl, 1, FoldConfig(rho=2, fold_k=2, d=d, fold_chain=[], negative=neg2))
    _, _, _, ok = ol.orc_fold(inner, ovl, 1, 2, d, 2, cfg.fold_poly, [], neg2, want_refold=False)
    assert ok == 0 and not res.assumption_ok


@pytest.mark.gpu
def test_gpu_fold_negative_zero_coefficients_take_the_exact_path():
    """A -0.0 coefficient (here the constant terms, where the reference's
    axpb(0, x, c0) leaf start yields -0 for negative x) switches the kernel to
    the operation-for-operation evaluation; still bit-exact with the oracle,
    including the signs of zeros."""
    from paper_2601_17561_b200.fold import FoldConfig, fold_stage
    rng = np.random.default_rng(9)
    d, blocks, batch, rho, fold_k = 128, 2, 2, 6, 3
    ovl = rng.integers(1, 100, size=(batch * rho, d * blocks)).astype(np.int32)
    inner = (rng.integers(-100, 101, size=ovl.shape) % (ovl + 1)).astype(np.int32)
    inner *= np.where(rng.random(ovl.shape) < 0.5, -1, 1).astype(np.int32)
    inner[:, ::7] = 0  # x = +-0 inputs
    fold_c = np.array([-0.0, 0.0, -0.0, 0.5, 0.0, -0.0, 0.25, -1.0])
    chain = [(0.0, np.array([-0.0, 1.0, -0.0, 0.0])), (0.0, np.array([-0.0, -0.0, 2.0]))]
    cfg = FoldConfig(rho=rho, fold_k=fold_k, d=d, fold_poly=fold_c, fold_chain=chain, negative=(-0.5, 0.5))
    res = fold_stage(inner, ovl, batch, cfg)
    st, f_o, r_o, ok = ol.orc_fold(inner, ovl, batch, rho, d, fold_k, fold_c, chain, (-0.5, 0.5))
    assert st == 0
    assert np.array_equal(res.folded.ravel().view(np.uint64), f_o.view(np.uint64))
    assert np.array_equal(res.refolded.ravel().view(np.uint64), r_o.view(np.uint64))
    assert res.assumption_ok == bool(ok)


@pytest.mark.gpu
def test_gpu_fold_empty_and_constant_polynomials():
    """An empty coefficient vector is the zero polynomial (degree 0, poly.cpp:10-15);
    a constant evaluates as axpb(0, x, c0) (poly.hpp:94)."""
    from paper_2601_17561_b200.fold import FoldConfig, fold_stage
    c = case("single")
    for fold_c in ([], [0.75], [0.0, 0.0, 0.0]):
        cfg = FoldConfig(rho=c["rho"], fold_k=c["fold_k"], d=c["d"], fold_poly=fold_c, fold_chain=c["chain"],
                         negative=c["neg"])
        res = fold_stage(c["inner"], c["overlap"], c["batch"], cfg)
        st, f_o, r_o, ok = ol.orc_fold(c["inner"], c["overlap"], c["batch"], c["rho"], c["d"], c["fold_k"],
                                       np.array(fold_c, np.float64), c["chain"], c["neg"])
        assert st == 0
        assert np.array_equal(res.folded.ravel().view(np.uint64), f_o.view(np.uint64))
        assert np.array_equal(res.refolded.ravel(), r_o)

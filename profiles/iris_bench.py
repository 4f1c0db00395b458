"""Times the plaintext iris scoring stage (irl_iris_match) at the paper's
scale: 7 * 2^14 templates, 32 eyes x 31 rotations, d = 2^14, host buffers in
and out (H2D of the packed templates inside the timed region).

    python profiles/iris_bench.py [--n-db 114688] [--eyes 32] [--rho 31] [--d 16384]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-db", type=int, default=7 << 14)
    ap.add_argument("--eyes", type=int, default=32)
    ap.add_argument("--rho", type=int, default=31)
    ap.add_argument("--d", type=int, default=1 << 14)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import ctypes as C
    from paper_2601_17561_b200 import capi
    from paper_2601_17561_b200.iris import pack_bits
    from paper_2601_17561_b200.modmat import default_context
    ctx = default_context()
    rng = np.random.default_rng(1)
    dc = pack_bits(rng.integers(0, 2, (a.n_db, a.d), dtype=np.uint8))
    dm = pack_bits((rng.random((a.n_db, a.d)) < 0.8).astype(np.uint8))
    qc = pack_bits(rng.integers(0, 2, (a.eyes, a.d), dtype=np.uint8))
    qm = pack_bits((rng.random((a.eyes, a.d)) < 0.8).astype(np.uint8))
    bits = np.zeros((a.eyes, a.n_db), np.uint8)
    res = np.zeros(a.eyes, np.int32)
    L = capi.lib()
    p = capi.ptr

    def run():
        st = L.irl_iris_match(ctx.handle, p(dc), p(dm), a.n_db, p(qc), p(qm), a.eyes, a.rho, a.d, 0.35, 1.0,
                              p(bits), p(res), None)
        assert st in (0, capi.IRL_ERR_ZERO_OVERLAP), st

    run()
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        run()
        ts.append(time.perf_counter() - t0)
    ms = float(np.median(ts) * 1e3)
    ops = 4.0 * a.n_db * a.eyes * a.rho * a.d  # two int8 GEMMs, 2 ops / MAC
    print(json.dumps({"stage": "iris_match one-shot (templates uploaded per call)", "n_db": a.n_db,
                      "cols": a.eyes * a.rho, "d": a.d, "ms_e2e": ms, "tops_e2e": ops / ms / 1e9,
                      "h2d_bytes": int(dc.nbytes * 2 + qc.nbytes * 2), "matches": int(bits.sum())}))
    # registered database: per query batch only the eyes' bits move
    from paper_2601_17561_b200.iris import IrisDatabase, Interval
    reg = IrisDatabase.from_packed(dc, dm, a.d, a.eyes * a.rho)
    reg.match_packed(qc, qm, a.eyes, a.rho, Interval(0.35, 1.0))
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        res2, bits2, _ = reg.match_packed(qc, qm, a.eyes, a.rho, Interval(0.35, 1.0))
        ts.append(time.perf_counter() - t0)
    ms2 = float(np.median(ts) * 1e3)
    assert (bits2 == bits).all() and (res2 == res).all()
    print(json.dumps({"stage": "iris_db_match per query batch (registered database)", "n_db": a.n_db,
                      "cols": a.eyes * a.rho, "d": a.d, "ms_e2e": ms2, "tops_e2e": ops / ms2 / 1e9,
                      "h2d_bytes": int(qc.nbytes * 2), "d2h_bytes": int(bits.nbytes)}))
    # CPU reference (unmodified iris::score, oracle/_ref) on a bounded sample:
    # 4 templates x all 992 query columns, one thread; extrapolated to the full DB
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
    import oracle_lib as ol
    if ol.ref_available():
        sample = 4
        unpack = lambda w, rows: np.unpackbits(w[:rows].view(np.uint8), axis=1, bitorder="little")[:, :a.d]  # noqa
        dcs, dms = unpack(dc, sample), unpack(dm, sample)
        qcs, qms = unpack(qc, a.eyes), unpack(qm, a.eyes)
        rc = np.zeros((a.eyes * a.rho, a.d), np.uint8)
        rm = np.zeros_like(rc)
        for e in range(a.eyes):
            for r in range(a.rho):
                idx = (np.arange(a.d) - r) % a.d
                rc[e * a.rho + r], rm[e * a.rho + r] = qcs[e][idx], qms[e][idx]
        t0 = time.perf_counter()
        ref = ol.ref_scores(rc, rm, dcs, dms)
        secs = time.perf_counter() - t0
        full = secs * a.n_db / sample
        print(json.dumps({"stage": "reference iris::score (oracle/_ref), 1 thread", "sample_templates": sample,
                          "sample_s": secs, "extrapolated_full_db_s": full,
                          "speedup_vs_registered_gpu": full * 1e3 / ms2,
                          "scores_finite": int(np.isfinite(ref).sum())}))


if __name__ == "__main__":
    main()

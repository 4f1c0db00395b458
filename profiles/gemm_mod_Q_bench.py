"""The reference's main entry point, gemm_mod_Q (modmat.cpp:162-195: residue
extraction, 24 per-modulus PPMMs, CRT lift), on BigMatrix operands of
46-byte entries mod Q: irl_gemm_mod_Q (host buffers in/out) against the
unmodified reference (oracle/_ref, one thread, as the reference runs it),
results compared byte for byte.

    python profiles/gemm_mod_Q_bench.py [--n 512]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    a = ap.parse_args()
    import oracle_lib as ol
    from paper_2601_17561_b200.modmat import build_paper_basis, gemm_mod_Q_le
    basis = build_paper_basis()
    p, e = basis.arrays()
    Q, w, n = basis.Q, basis.width(), a.n
    rng = np.random.default_rng(3)
    def rand_le(count):
        x = rng.integers(0, 256, (count, w), dtype=np.uint8)
        x[:, -1] = 0  # < 2^360 < Q
        return x
    A, B = rand_le(n * n), rand_le(n * n)
    gemm_mod_Q_le(A[:64], B[:64], 8, 8, 8, w, basis)  # warm-up
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        C = gemm_mod_Q_le(A, B, n, n, n, w, basis)
        ts.append(time.perf_counter() - t0)
    gpu_ms = float(np.median(ts) * 1e3)
    rec = {"call": "gemm_mod_Q (irl_gemm_mod_Q, host BigMatrix buffers)", "m=k=n": n, "moduli": len(p),
           "gpu_e2e_ms": gpu_ms, "int8_tops_e2e": 6.0 * len(p) * n ** 3 / gpu_ms / 1e9}
    if ol.ref_available():
        Cr = np.zeros_like(C)
        t0 = time.perf_counter()
        st = ol.ref().ref_gemm_mod_Q(ol.ptr(A, ol.u8p), ol.ptr(B, ol.u8p), ol.ptr(Cr, ol.u8p), n, n, n, w,
                                     ol.ptr(p, ol.u32p), ol.ptr(e, ol.u32p), len(p))
        cpu_s = time.perf_counter() - t0
        assert st == 0
        rec.update({"reference_s": cpu_s, "reference_threads": 1, "speedup": cpu_s * 1e3 / gpu_ms,
                    "bit_exact": bool((Cr == C).all())})
    print(json.dumps(rec))


if __name__ == "__main__":
    main()

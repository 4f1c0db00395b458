"""BASELINE configs[0] (c1): single-limb PPMM mod 127^2 (digit split + 3 int8
GEMMs), A 256 x 4096 by B 4096 x 4096 uniform residues -> C 256 x 4096.
Times the reference-API call irl_gemm_mod_psq (host int32 buffers in/out,
i.e. gemm_mod_psq, modmat.cpp:143-160) on the B200 and the unmodified
reference gemm_mod_psq (oracle/_ref) on one host thread, and checks the two
results are identical.

    python profiles/c1_bench.py
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import oracle_lib as ol
    from paper_2601_17561_b200 import modmat
    p, m, k, n = 127, 256, 4096, 4096
    rng = np.random.default_rng(1)
    a = rng.integers(0, p * p, (m, k), dtype=np.int32)
    b = rng.integers(0, p * p, (k, n), dtype=np.int32)
    c = modmat.gemm_mod_psq(a, b, p)  # warm-up (context, kernels)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        c = modmat.gemm_mod_psq(a, b, p)
        ts.append(time.perf_counter() - t0)
    gpu_ms = float(np.median(ts) * 1e3)
    # the same call with page-locked inputs (a caller's pinned buffers): the C ABI
    # DMAs them directly instead of staging through its bounce buffers
    import torch
    ap = torch.from_numpy(a).pin_memory().numpy()
    bp = torch.from_numpy(b).pin_memory().numpy()
    modmat.gemm_mod_psq(ap, bp, p)
    tp = []
    for _ in range(10):
        t0 = time.perf_counter()
        cp = modmat.gemm_mod_psq(ap, bp, p)
        tp.append(time.perf_counter() - t0)
    assert (np.asarray(cp) == np.asarray(c)).all()
    ops = 6.0 * m * n * k
    rec = {"config": "c1: gemm_mod_psq mod 127^2, 256x4096 . 4096x4096", "gpu_e2e_ms": gpu_ms,
           "gpu_e2e_ms_pinned_inputs": float(np.median(tp) * 1e3),
           "gpu_e2e_tops": ops / gpu_ms / 1e9, "h2d_bytes": int(a.nbytes + b.nbytes), "d2h_bytes": int(c.nbytes)}
    if ol.ref_available():
        cc = np.zeros((m, n), np.int32)
        t0 = time.perf_counter()
        st = ol.ref().ref_gemm_mod_psq(ol.ptr(a, ol.i32p), ol.ptr(b, ol.i32p), ol.ptr(cc, ol.i32p), m, k, n, p)
        cpu_s = time.perf_counter() - t0
        assert st == 0
        rec.update({"cpu_reference_s": cpu_s, "cpu_reference_threads": 1, "cpu_kind": "reference (oracle/_ref)",
                    "speedup_e2e": cpu_s * 1e3 / gpu_ms, "bit_exact": bool((cc == np.asarray(c)).all())})
    print(json.dumps(rec))


if __name__ == "__main__":
    main()

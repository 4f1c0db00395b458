"""irl_ccmm_run at c4 with pageable vs page-locked host buffers (the
reference-facing C++ mirror passes std::vector storage, i.e. pageable).

    python profiles/e2e_pageable.py [--parts 8]
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
    ap.add_argument("--parts", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, synth_query
    M, K, N = 1 << 14, 24576, 992
    eng = CcmmEngine(parts=a.parts, m=M, k=K, max_n=N)
    eng.synth_db(seed=1)
    q = synth_query(2, K, N, eng.moduli)
    out = np.empty((a.parts, eng.nmod, N, M), np.uint16)
    qp = torch.from_numpy(q.view(np.int16)).pin_memory().numpy().view(np.uint16)
    op = torch.empty(out.shape, dtype=torch.int16).pin_memory().numpy().view(np.uint16)
    res = {}
    for name, qq, oo in (("pinned", qp, op), ("pageable", q, out), ("pinned", qp, op), ("pageable", q, out)):
        eng.run(qq, oo)
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            eng.run(qq, oo)
            ts.append((time.perf_counter() - t0) * 1e3)
        res.setdefault(name, []).append(round(min(ts), 2))
    assert (out == op).all()
    print(json.dumps({"parts": a.parts, "e2e_ms": res}))


if __name__ == "__main__":
    main()

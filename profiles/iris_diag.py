"""FP4 iris match kernel diagnostics at the paper's scale (7 * 2^14 templates,
d = 2^14, 32 x 31 columns): the kernel's per-pair cycle counters for the main
(960-column, 1x4-cluster) launch, as profiles/ppmm_diag.py does for the PPMM.

    python profiles/iris_diag.py [--runs 3]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=3)
    ap.add_argument("--inner", action="store_true", help="the fold path's raw inner-product / overlap launch")
    a = ap.parse_args()
    from paper_2601_17561_b200 import capi
    from paper_2601_17561_b200.iris import Interval, IrisDatabase
    d, n_db, eyes, rho = 1 << 14, 7 << 14, 32, 31
    rng = np.random.default_rng(5)
    words = d // 64
    bits = lambda n: rng.integers(0, 1 << 63, size=(n, words), dtype=np.uint64)  # noqa: E731
    dc, dm, qc, qm = bits(n_db), bits(n_db) | bits(n_db), bits(eyes), bits(eyes) | bits(eyes)
    db = IrisDatabase.from_packed(dc, dm, d, eyes * rho)
    L = capi.lib()
    h = db.ctx.handle
    from paper_2601_17561_b200.fold import FoldConfig
    cfg = FoldConfig(rho=rho, fold_k=16, d=d)

    def call():
        if a.inner:  # the fold path: inner products and overlaps (kModeInnerF4), then the fold stage
            db.fold_packed(qc, qm, eyes, cfg, want_folded=True, want_refolded=False)
        else:
            db.match_packed(qc, qm, eyes, rho, Interval(0.35, 1.0))
    call()
    L.irl_diag_ppmm(h, 1, None, 0)
    buf = (C.c_uint64 * (1024 * 16))()
    for _ in range(a.runs):
        call()
        L.irl_diag_ppmm(h, 1, buf, len(buf))
        st = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16).astype(np.float64)
        act = st[:, 4] > 0
        for name, sel in (("main cluster pairs", np.arange(1024) < 60), ("filler pairs", np.arange(1024) >= 60)):
            g = st[act & sel]
            if len(g):
                c = g[:, 4]
                print(json.dumps({"group": name, "pairs": len(g),
                                  "mma_full_wait_pct": float(np.mean(g[:, 2] / c) * 100),
                                  "mma_tmem_wait_pct": float(np.mean(g[:, 3] / c) * 100),
                                  "producer_empty_wait_pct": float(np.mean(g[:, 0] / c) * 100),
                                  "epi_busy_pct": float(np.mean(g[:, 6] / c) * 100),
                                  "tiles": [int(g[:, 11].min()), int(g[:, 11].max())]}))
        s = st[act]
        ns = s[:, 8] - s[:, 7]
        cyc = s[:, 4]
        print(json.dumps({
            "pairs": int(act.sum()),
            "kernel_ms": float((s[:, 8].max() - s[:, 7].min()) / 1e6),
            "clock_mhz": float(np.mean(cyc / ns * 1e3)),
            "mma_full_wait_pct": float(np.mean(s[:, 2] / cyc) * 100),
            "mma_tmem_wait_pct": float(np.mean(s[:, 3] / cyc) * 100),
            "producer_gate_pct": float(np.mean(s[:, 1] / cyc) * 100),
            "producer_empty_wait_pct": float(np.mean(s[:, 0] / cyc) * 100),
            "epi_busy_pct": float(np.mean(s[:, 6] / cyc) * 100),
            "epi_wait_pct": float(np.mean(s[:, 5] / cyc) * 100),
            "tiles_min_max": [int(s[:, 11].min()), int(s[:, 11].max())],
            "pair_ms_min_max": [float(ns.min() / 1e6), float(ns.max() / 1e6)],
        }), flush=True)
    L.irl_diag_ppmm(h, 0, None, 0)
    db.close()


if __name__ == "__main__":
    main()

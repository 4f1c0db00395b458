"""Times the Alg. 2 fold stage (csrc/fold.cu) at the paper's scale: products
and overlaps of 32 eyes x 31 rotations against 7 * 2^14 templates (d = 2^14,
blocks = 7, fold_k = 16: two rotation groups), published folding polynomial,
a 3-stage fold chain (degrees 15, 31, 3).

* kernel: irl_fold_stage_device on device-resident inner / overlap (CUDA
  events on the launching stream, 20 launches), against the HBM roofline:
  algorithmic bytes = 8 B per (column, template) read + 8 B per output
  element written;
* e2e: IrisDatabase.fold (irl_iris_db_fold): query bits H2D, the two int8
  GEMMs, the fold stage, folded + refolded D2H.

    python profiles/fold_bench.py [--folded]
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
    ap.add_argument("--folded", action="store_true", help="also write the per-group folded messages")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch

    import oracle_lib as ol  # stand-in fold chain coefficients only
    from paper_2601_17561_b200.fold import FoldConfig, fold_stage_device
    from paper_2601_17561_b200.iris import IrisDatabase

    d, n_db, eyes, rho, fold_k = 1 << 14, 7 << 14, 32, 31, 16
    cols, blocks, groups = eyes * rho, n_db // d, -(-rho // fold_k)
    cfg = FoldConfig(rho=rho, fold_k=fold_k, d=d, fold_chain=ol.fold_chain_for_tests("wide"), negative=(-0.05, 0.05))
    g = torch.Generator(device="cuda").manual_seed(1)
    ovl = torch.randint(1, d, (cols, n_db), dtype=torch.int32, device="cuda", generator=g)
    inner = (torch.rand((cols, n_db), device="cuda", generator=g) * (2 * ovl + 1)).to(torch.int32) - ovl
    folded = torch.empty(eyes * blocks * groups * d, dtype=torch.float64, device="cuda") if a.folded else None
    refolded = torch.empty(eyes * blocks * d, dtype=torch.float64, device="cuda")
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(3):
        fold_stage_device(inner, ovl, eyes, cfg, folded, refolded, flags)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(a.reps):
        fold_stage_device(inner, ovl, eyes, cfg, folded, refolded, flags)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    out_elems = eyes * blocks * d * (1 + (groups if a.folded else 0))
    nbytes = 8 * cols * n_db + 8 * out_elems
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    kernel = {"kernel": "fold_stage_kernel", "ms": ms, "bytes": nbytes, "GB/s": nbytes / ms / 1e6,
              "hbm_frac": nbytes / ms / 1e6 / peaks["hbm_gbs"], "pairs": cols * n_db,
              "poly_evals": cols * n_db + 3 * eyes * blocks * groups * d}

    # e2e from templates on a registered database
    rng = np.random.default_rng(2)
    words = d // 64
    bits = lambda n: rng.integers(0, 1 << 63, size=(n, words), dtype=np.uint64)  # noqa: E731
    dc, dm, qc, qm = bits(n_db), bits(n_db) | bits(n_db), bits(eyes), bits(eyes) | bits(eyes)
    db = IrisDatabase.from_packed(dc, dm, d, max_cols=cols)
    from paper_2601_17561_b200.fold import shapes
    fshape, rshape = shapes(cfg, eyes, n_db)

    def timed(**outs):
        db.fold_packed(qc, qm, eyes, cfg, want_folded=a.folded, **outs)
        ts = []
        for _ in range(7):
            t0 = time.perf_counter()
            db.fold_packed(qc, qm, eyes, cfg, want_folded=a.folded, **outs)
            ts.append((time.perf_counter() - t0) * 1e3)
        return sorted(ts)[len(ts) // 2]

    def pinned(shape):
        return torch.zeros(tuple(shape), dtype=torch.float64).pin_memory().numpy()
    e2e = {"fresh_output_arrays": timed(),
           "reused_pageable_outputs": timed(out_folded=np.zeros(fshape) if a.folded else None,
                                            out_refolded=np.zeros(rshape)),
           "reused_pinned_outputs": timed(out_folded=pinned(fshape) if a.folded else None,
                                          out_refolded=pinned(rshape))}
    ts = [e2e["fresh_output_arrays"]]
    db.close()
    rec = {"workload": f"Alg. 2 fold stage: {eyes} eyes x {rho} rotations vs {n_db} templates, d={d}, "
                       f"fold_k={fold_k}, chain degrees 15/31/3", "fold_kernel": kernel,
           "e2e_iris_db_fold_ms": float(np.median(ts)), "e2e_ms_by_output_buffers": e2e,
           "e2e_note": "query bits H2D + the two FP4 products (inner, overlap) + fold stage + outputs D2H"}
    print(json.dumps(rec))


if __name__ == "__main__":
    main()

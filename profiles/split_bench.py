"""Times the per-step query split (split_cols_u16_vec_kernel) alone at the c4
query geometry: 24 moduli x K = 24576 x N = 992 uint16 residues -> int8
digit planes; 4 B of HBM traffic per (entry, modulus).

    python profiles/split_bench.py [--n 992] [--k 24576] [--reps 20]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=992)
    ap.add_argument("--k", type=int, default=24576)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import os
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query
    eng = CcmmEngine(parts=1, m=256, k=a.k, max_n=a.n)
    q_dev, _ = staging_tensors(eng, a.n)
    q_dev.copy_(torch.from_numpy(synth_query(2, a.k, a.n, eng.moduli).view(np.int16)))
    s = torch.cuda.Stream()
    for _ in range(3):
        eng.run_device(None, a.n, None, nparts=0, stream=s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.reps):
        eng.run_device(None, a.n, None, nparts=0, stream=s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    by = 4.0 * eng.nmod * a.k * a.n
    print(json.dumps({"tile": os.environ.get("IRL_SPLIT_TILE", "default"), "ms": ms, "GBps": by / ms / 1e6}))


if __name__ == "__main__":
    main()

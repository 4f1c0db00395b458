"""Times irl_ccmm_rescale (f2 ModDown, drop 3, rounding) over one c4 part's
outputs (24 moduli x 992 x 2^14 residues) in isolation.

    python profiles/moddown_bench.py [--reps 10]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--drop", type=int, default=3)
    a = ap.parse_args()
    import os

    import numpy as np
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query
    N, M = 992, 1 << 14
    eng = CcmmEngine(parts=1, m=M, k=128, max_n=N)
    eng.synth_db(1)
    qd, _ = staging_tensors(eng, N)
    qd.copy_(torch.from_numpy(synth_query(2, 128, N, eng.moduli).view(np.int16)))
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    eng.run_device(None, N, None, stream=s.cuda_stream)  # valid residues in the engine outputs
    dst = torch.empty((1, eng.nmod - a.drop, N, M), dtype=torch.int16, device="cuda")
    for _ in range(2):
        eng.rescale(N, dst, a.drop, True, stream=s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.reps):
        eng.rescale(N, dst, a.drop, True, stream=s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    by = 2.0 * (2 * eng.nmod - a.drop) * N * M
    kern = "rescale_vec_kernel (folded 64-bit)" if os.environ.get("IRL_RESCALE_FOLDED") else "rescale_r_kernel"
    print(json.dumps({"kernel": kern, "ms": ms, "GBps": by / ms / 1e6, "bytes": by}))


if __name__ == "__main__":
    main()

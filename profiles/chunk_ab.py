"""Same-process A/B of e2e modulus-chunk plans (IRL_E2E_CHUNKS) for irl_ccmm_run
at the c4 geometry: plans alternate within one engine, so box and clock drift
hit every plan alike.

    python profiles/chunk_ab.py [--parts 8] [--reps 8] [--plans default,3:21,4:20]
"""
import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", type=int, default=8)
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--plans", default="default,3:21,4:20,2:22,1:6:17")
    a = ap.parse_args()
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, synth_query
    N, M, K = 992, 1 << 14, 24576
    eng = CcmmEngine(parts=a.parts, m=M, k=K, max_n=N)
    eng.synth_db(1)
    q = torch.from_numpy(synth_query(2, K, N, eng.moduli).view(np.int16)).pin_memory().numpy().view(np.uint16)
    out = torch.empty((a.parts, eng.nmod, N, M), dtype=torch.int16).pin_memory().numpy().view(np.uint16)
    plans = a.plans.split(",")
    res = {p: [] for p in plans}
    eng.run(q, out)
    for _ in range(a.reps):
        for p in plans:
            if p == "default":
                os.environ.pop("IRL_E2E_CHUNKS", None)
            else:
                os.environ["IRL_E2E_CHUNKS"] = p.replace(":", ",")
            t0 = time.perf_counter()
            eng.run(q, out)
            res[p].append((time.perf_counter() - t0) * 1e3)
    os.environ.pop("IRL_E2E_CHUNKS", None)
    print(json.dumps({"parts": a.parts, "median_ms": {p: round(statistics.median(v), 2) for p, v in res.items()},
                      "all_ms": {p: [round(x, 1) for x in v] for p, v in res.items()}}))


if __name__ == "__main__":
    main()

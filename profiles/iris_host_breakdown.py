"""Where the host-to-host time of the registered-database iris match goes:
the full call (match bits to a pageable numpy buffer), the same into pinned
memory, and without match bits (first-event results only). Paper scale.

    python profiles/iris_host_breakdown.py [--reps 30]
"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    import torch
    from paper_2601_17561_b200 import capi
    from paper_2601_17561_b200.iris import IrisDatabase, _p
    d, n_db, eyes, rho = 1 << 14, 7 << 14, 32, 31
    rng = np.random.default_rng(5)
    words = d // 64
    bits = lambda n: rng.integers(0, 1 << 63, size=(n, words), dtype=np.uint64)  # noqa: E731
    dc, dm, qc, qm = bits(n_db), bits(n_db) | bits(n_db), bits(eyes), bits(eyes) | bits(eyes)
    db = IrisDatabase.from_packed(dc, dm, d, eyes * rho)
    L = capi.lib()
    res = np.zeros(eyes, np.int32)
    pageable = np.zeros((eyes, n_db), np.uint8)
    pinned = torch.zeros((eyes, n_db), dtype=torch.uint8).pin_memory().numpy()
    out = {}
    for name, buf in (("bits_pageable", pageable), ("bits_pinned", pinned), ("no_bits", None)):
        ts = []
        for i in range(a.reps + 3):
            t0 = time.perf_counter()
            L.irl_iris_db_match(db.handle, _p(qc), _p(qm), eyes, rho, 0.35, 1.0, _p(buf), _p(res), None)
            if i >= 3:
                ts.append((time.perf_counter() - t0) * 1e3)
        out[name] = round(statistics.median(ts), 4)
    print(json.dumps({"ms_median": out}), flush=True)
    db.close()


if __name__ == "__main__":
    main()

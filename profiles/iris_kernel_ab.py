"""Times the iris product GEMM alone (kModeInner / kModeInnerF4 through
irl_iris_db_fold's GEMM, CUDA events around irl_iris_inner_overlap's device
part is not exposed, so this times IrisDatabase.match_packed end to end and
the fold path) for A/B of plane formats and cluster shapes via env knobs.

    IRL_IRIS_I8=1 IRL_PPMM_CLUSTER=1x1 python profiles/iris_kernel_ab.py
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    from paper_2601_17561_b200.iris import IrisDatabase, Interval
    d, n_db, eyes, rho = 1 << 14, 7 << 14, 32, 31
    rng = np.random.default_rng(1)
    words = d // 64
    bits = lambda n: rng.integers(0, 1 << 63, size=(n, words), dtype=np.uint64)  # noqa: E731
    dc, dm, qc, qm = bits(n_db), bits(n_db) | bits(n_db), bits(eyes), bits(eyes) | bits(eyes)
    db = IrisDatabase.from_packed(dc, dm, d, eyes * rho)
    db.match_packed(qc, qm, eyes, rho, Interval(0.35, 1.0))
    ts = []
    for _ in range(int(os.environ.get("REPS", "9"))):
        t0 = time.perf_counter()
        db.match_packed(qc, qm, eyes, rho, Interval(0.35, 1.0))
        ts.append((time.perf_counter() - t0) * 1e3)
    print(json.dumps({"iris_i8": bool(os.environ.get("IRL_IRIS_I8")), "cluster": os.environ.get("IRL_PPMM_CLUSTER"),
                      "match_ms_median": round(float(np.median(ts)), 3), "match_ms_min": round(float(np.min(ts)), 3), "p25": round(float(np.percentile(ts, 25)), 3)}))
    db.close()


if __name__ == "__main__":
    main()

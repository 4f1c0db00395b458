"""Registered-database iris match at the paper's scale (7 * 2^14 templates of
d = 2^14, 32 eyes x 31 rotations), host query bits in, match bits out: median
of --reps calls. Run once per setting of an environment knob (IRL_IRIS_I8,
IRL_IRIS_NO_SPLIT) and alternate processes for an A/B.

    IRL_IRIS_I8=1 python profiles/iris_match_ab.py [--reps 20]
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
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--check", action="store_true", help="compare bits with a one-shot int8 run")
    a = ap.parse_args()
    from paper_2601_17561_b200.iris import Interval, IrisDatabase
    d, n_db, eyes, rho = 1 << 14, 7 << 14, 32, 31
    rng = np.random.default_rng(5)
    words = d // 64
    bits = lambda n: rng.integers(0, 1 << 63, size=(n, words), dtype=np.uint64)  # noqa: E731
    dc, dm, qc, qm = bits(n_db), bits(n_db) | bits(n_db), bits(eyes), bits(eyes) | bits(eyes)
    dc[100] = np.roll(qc[31], 0)
    dm[100] = qm[31]
    db = IrisDatabase.from_packed(dc, dm, d, eyes * rho)
    out = np.zeros((eyes, n_db), np.uint8) if os.environ.get("IRL_AB_FRESH_BITS") is None else None
    for _ in range(3):
        res, b, _ = db.match_packed(qc, qm, eyes, rho, Interval(0.35, 1.0), out_bits=out)
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        res, b, _ = db.match_packed(qc, qm, eyes, rho, Interval(0.35, 1.0), out_bits=out)
        ts.append((time.perf_counter() - t0) * 1e3)
    digest = int(np.bitwise_xor.reduce(np.packbits(b).view(np.uint8)))
    print(json.dumps({"no_split": bool(os.environ.get("IRL_IRIS_NO_SPLIT")), "i8": bool(os.environ.get("IRL_IRIS_I8")),
                      "ms_median": statistics.median(ts), "ms_min": min(ts), "matches": int(b.sum()),
                      "res": res.tolist()[-2:], "bits_xor": digest}), flush=True)
    db.close()


if __name__ == "__main__":
    main()

"""f3 ingest throughput: one DB part (2^14 templates x K = 24576 entries mod Q,
46 bytes each = 18.5 GB) streamed from the reference's BigMatrix file format
into int8 digit planes (irl_ccmm_load_part_file: double-buffered file read,
H2D and residue/digit split). The file is written first (so the second load
reads from the page cache) and removed afterwards.

    python profiles/ingest_bench.py [--rows 16384] [--dir /tmp]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1 << 14)
    ap.add_argument("--k", type=int, default=24576)
    ap.add_argument("--dir", default="/tmp")
    ap.add_argument("--file", default=None, help="load this existing BigMatrix file (not written, not removed)")
    ap.add_argument("--keep", action="store_true", help="keep the written file (print its path)")
    a = ap.parse_args()
    from paper_2601_17561_b200.ccmm import CcmmEngine
    eng = CcmmEngine(parts=1, m=a.rows, k=a.k, max_n=32)
    Q = eng.basis.Q
    width = (Q.bit_length() + 7) // 8
    path = Path(a.file) if a.file else Path(a.dir) / f"irl_ingest_{os.getpid()}.bin"
    rng = np.random.default_rng(5)
    t0 = time.perf_counter()
    with open(os.devnull if a.file else path, "wb") as f:
        f.write(f"{a.rows} {a.k} {Q}\n".encode())
        rows_per = max(1, (256 << 20) // (a.k * width))
        for r0 in range(0, 0 if a.file else a.rows, rows_per):
            nr = min(rows_per, a.rows - r0)
            ent = rng.integers(0, 256, (nr * a.k, width), dtype=np.uint8)
            ent[:, -1] = 0
            f.write(ent.tobytes())
    write_s = time.perf_counter() - t0
    size = path.stat().st_size
    res = []
    for _ in range(2):
        t0 = time.perf_counter()
        eng.load_part_file(0, path)
        res.append(time.perf_counter() - t0)
    if not (a.file or a.keep):
        path.unlink()
    print(json.dumps({"bytes": size, "write_s": write_s, "load_s": res, "readers": os.environ.get("IRL_INGEST_READERS", "4"),
                      "file": str(path) if a.keep else None,
                      "load_GBps": [size / t / 1e9 for t in res],
                      "entries_per_s": [a.rows * a.k / t for t in res]}))


if __name__ == "__main__":
    main()

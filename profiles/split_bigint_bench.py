"""Times the mod-Q ingest kernel (irl_split_bigint: 46-byte entries ->
residues mod 24 p^2 -> centred int8 digit planes) on device-resident entries,
the DB layout (transpose = 0) of a 2048 x 24576 block, and reports its HBM
rate against the algorithmic 46 B read + 2 * 24 B written per entry.

    python profiles/split_bigint_bench.py [--rows 2048] [--reps 5]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=2048)
    ap.add_argument("--cols", type=int, default=24576)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import ctypes as C

    import torch
    from paper_2601_17561_b200 import capi
    from paper_2601_17561_b200.modmat import build_paper_basis, default_context
    ctx = default_context()
    b = build_paper_basis()
    p, e = b.arrays()
    w = b.width()
    n = a.rows * a.cols
    g = torch.Generator(device="cuda").manual_seed(1)
    ent = torch.randint(0, 256, (n, w), dtype=torch.uint8, device="cuda", generator=g)
    ent[:, -1] = 0  # below 2^360 < Q
    ldk = (a.cols + 15) // 16 * 16
    planes = torch.empty((len(p), 2, a.rows, ldk), dtype=torch.int8, device="cuda")
    s = torch.cuda.Stream()

    def run():
        ctx.check(capi.lib().irl_split_bigint(ctx.handle, C.c_void_p(ent.data_ptr()), w, a.rows, a.cols, 0,
                                               capi.ptr(p, capi.u32p), capi.ptr(e, capi.u32p), len(p),
                                               C.c_void_p(planes.data_ptr()), ldk, C.c_void_p(s.cuda_stream)))
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.reps):
        run()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    by = n * (w + 2 * len(p))
    print(json.dumps({"kernel": "split_bigint", "entries": n, "width": w, "ms": ms, "GBps": by / ms / 1e6,
                      "entries_per_s": n / ms * 1e3, "bytes": by}))


if __name__ == "__main__":
    main()

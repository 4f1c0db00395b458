"""PPMM kernel diagnostics: where the MMA issuer and the producers wait.

    python profiles/ppmm_diag.py [--parts 8] [--rows 16384] [--k 24576] [--n 992]

Runs the CCMM engine with the kernel's cycle counters on (irl_diag_ppmm) and
prints per-pair averages: MMA full-barrier waits (data late), TMEM-empty waits
(epilogue late), producer gate/empty waits, epilogue busy time, and the
effective SM clock (clock64 cycles / globaltimer ns).
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
    ap.add_argument("--parts", type=int, default=8)
    ap.add_argument("--rows", type=int, default=1 << 14)
    ap.add_argument("--k", type=int, default=24576)
    ap.add_argument("--n", type=int, default=992)
    ap.add_argument("--runs", type=int, default=3)
    a = ap.parse_args()
    import torch
    from paper_2601_17561_b200 import capi
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query

    eng = CcmmEngine(parts=a.parts, m=a.rows, k=a.k, max_n=a.n)
    eng.synth_db(1)
    q_dev, _ = staging_tensors(eng, a.n)
    q_dev.copy_(torch.from_numpy(synth_query(2, a.k, a.n, eng.moduli).view(np.int16)))
    torch.cuda.synchronize()
    L = capi.lib()
    eng.run_device(None, a.n, None, part0=0, nparts=0)
    L.irl_diag_ppmm(eng.ctx.handle, 1, None, 0)
    buf = (C.c_uint64 * (1024 * 16))()
    rows = []
    for _ in range(a.runs):
        eng.run_device(None, a.n, None, q_ready=True)
        L.irl_diag_ppmm(eng.ctx.handle, 1, buf, len(buf))
        st = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16).astype(np.float64)
        act = st[:, 4] > 0
        s = st[act]
        ns = s[:, 8] - s[:, 7]
        cyc = s[:, 4]
        rows.append({
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
            "slowest_pairs": [(int(i), round(float((st[i, 8] - st[i, 7]) / 1e6), 2))
                              for i in np.argsort(-(st[:, 8] - st[:, 7]) * act)[:6]],
            "pair_ms_by_id": [round(float(x / 1e6), 1) for x in (st[:, 8] - st[:, 7])[act]],
            "smid_by_pair": [int(x) for x in st[:, 12][act]],
        })
    L.irl_diag_ppmm(eng.ctx.handle, 0, None, 0)
    ops = 6.0 * eng.nmod * a.rows * a.n * a.k * a.parts
    for r in rows:
        r["tops"] = ops / (r["kernel_ms"] * 1e-3) / 1e12
        print(json.dumps(r))


if __name__ == "__main__":
    main()

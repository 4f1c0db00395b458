"""BASELINE configs[4] on one B200: query batch 32 -> 256 eyes (x 31
rotations) against one slice of 2^14 -> 2^17 templates, K = 24576, 24 moduli.
Device-resident PPMM timing (CUDA events on the engine stream) for every
point whose engine fits in HBM with the full batch staged, plus the e2e
column-chunked run (irl_ccmm_run, host buffers) at the corner that does not.

    python profiles/c5_sweep.py [--eyes 32,64,128,256] [--rows 14,15,16,17]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
HBM_BUDGET = 170e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--eyes", default="32,64,128,256")
    ap.add_argument("--rows", default="14,15,16,17")
    ap.add_argument("--k", type=int, default=24576)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--corner-e2e", action="store_true")
    a = ap.parse_args()
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query
    nmod, K = 24, a.k
    for lg in map(int, a.rows.split(",")):
        M = 1 << lg
        for eyes in map(int, a.eyes.split(",")):
            N = eyes * 31
            need = nmod * 2 * M * K + 2 * nmod * K * N * 2 + nmod * N * M * 2
            rec = {"templates": M, "eyes": eyes, "N": N, "K": K, "hbm_bytes": need}
            if need > HBM_BUDGET:
                rec["skipped"] = "does not fit with the whole batch staged; see the e2e corner run"
                print(json.dumps(rec), flush=True)
                continue
            eng = CcmmEngine(parts=1, m=M, k=K, max_n=N)
            eng.synth_db(1)
            q_dev, _ = staging_tensors(eng, N)
            q_dev.copy_(torch.from_numpy(synth_query(2, K, N, eng.moduli).view(np.int16)))
            torch.cuda.synchronize()
            s = torch.cuda.Stream()
            eng.run_device(None, N, None, stream=s.cuda_stream)
            eng.run_device(None, N, None, q_ready=True, stream=s.cuda_stream)
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                eng.run_device(None, N, None, q_ready=True, stream=s.cuda_stream)
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            ops = 6.0 * nmod * M * N * K
            rec.update({"ppmm_ms": ms, "tops": ops / ms / 1e9})
            print(json.dumps(rec), flush=True)
            eng.close()
            del q_dev
            torch.cuda.empty_cache()
    if a.corner_e2e:
        M, eyes = 1 << 17, 256
        N = eyes * 31
        eng = CcmmEngine(parts=1, m=M, k=K, max_n=1024)
        eng.synth_db(1)
        q = torch.from_numpy(synth_query(2, K, N, eng.moduli).view(np.int16)).pin_memory().numpy().view(np.uint16)
        out = torch.empty((1, nmod, N, M), dtype=torch.int16).pin_memory().numpy().view(np.uint16)
        eng.run(q[:, :, :1024].copy(), np.empty((1, nmod, 1024, M), np.uint16))  # warm-up (lazy init)
        t0 = time.perf_counter()
        eng.run(q, out)
        sec = time.perf_counter() - t0
        ops = 6.0 * nmod * M * N * K
        print(json.dumps({"templates": M, "eyes": eyes, "N": N, "K": K, "e2e_s": sec, "e2e_tops": ops / sec / 1e12,
                          "column_chunk": 1024, "d2h_bytes": int(out.nbytes)}), flush=True)


if __name__ == "__main__":
    main()

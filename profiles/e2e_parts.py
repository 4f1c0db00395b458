"""e2e (irl_ccmm_run, pinned host buffers) of the c4 query batch against 1, 2,
4 and 8 parts on one GPU: the per-GPU e2e of the 8/4/2/1-GPU layouts.

    python profiles/e2e_parts.py [--parts 1,2,4,8]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", default="1,2,4,8")
    a = ap.parse_args()
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query
    N, M, K = 992, 1 << 14, 24576
    for parts in map(int, a.parts.split(",")):
        eng = CcmmEngine(parts=parts, m=M, k=K, max_n=N)
        eng.synth_db(1)
        qh = synth_query(2, K, N, eng.moduli)
        q = torch.from_numpy(qh.view(np.int16)).pin_memory().numpy().view(np.uint16)
        out = torch.empty((parts, eng.nmod, N, M), dtype=torch.int16).pin_memory().numpy().view(np.uint16)
        eng.run(q, out)
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            eng.run(q, out)
            ts.append(time.perf_counter() - t0)
        # device-resident step for comparison
        qd, _ = staging_tensors(eng, N)
        qd.copy_(torch.from_numpy(qh.view(np.int16)))
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng.run_device(None, N, None, stream=s.cuda_stream)
        e0.record(s)
        for _ in range(4):
            eng.run_device(None, N, None, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        print(json.dumps({"parts": parts, "e2e_ms": [round(t * 1e3, 2) for t in ts],
                          "device_ms": round(e0.elapsed_time(e1) / 4, 2)}), flush=True)
        eng.close()
        del out, q


if __name__ == "__main__":
    main()

"""Per-chunk timeline of the e2e CCMM call (irl_ccmm_run, host buffers) at the
c4 workload: IRL_E2E_TRACE=1 makes the C ABI print H2D / PPMM / D2H
completion times per modulus chunk.

    IRL_E2E_TRACE=1 python profiles/e2e_trace.py
"""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    os.environ.setdefault("IRL_E2E_TRACE", "1")
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, synth_query
    N, M, K = 992, 1 << 14, 24576
    eng = CcmmEngine(parts=8, m=M, k=K, max_n=N)
    eng.synth_db(1)
    q = torch.from_numpy(synth_query(2, K, N, eng.moduli).view(np.int16)).pin_memory().numpy().view(np.uint16)
    out = torch.empty((8, eng.nmod, N, M), dtype=torch.int16).pin_memory().numpy().view(np.uint16)
    for it in range(3):
        t0 = time.perf_counter()
        eng.run(q, out)
        print(f"e2e run {it}: {(time.perf_counter() - t0) * 1e3:.1f} ms", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()

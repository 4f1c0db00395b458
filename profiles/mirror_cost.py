"""Cost of the fused a-part exchange in the owner's GEMM: one part (the 8-GPU
owner's share) with 0 vs 7 mirror buffers. The mirrors are local buffers
here (one GPU), so this measures the epilogue's extra stores and HBM writes,
not NVLink.

    python profiles/mirror_cost.py
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query
    N, M, K = 992, 1 << 14, 24576
    eng = CcmmEngine(parts=1, m=M, k=K, max_n=N)
    eng.synth_db(1)
    qd, od = staging_tensors(eng, N)
    qd.copy_(torch.from_numpy(synth_query(2, K, N, eng.moduli).view(np.int16)))
    torch.cuda.synchronize()
    mirrors = [torch.empty((eng.nmod, N, M), dtype=torch.int16, device="cuda") for _ in range(7)]
    s = torch.cuda.Stream()
    eng.run_device(None, N, None, stream=s.cuda_stream)

    def timed(k, reps=10):
        eng.set_mirror_ptrs(0, N, mirrors[:k])
        for _ in range(2):
            eng.run_device(None, N, None, q_ready=True, stream=s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            eng.run_device(None, N, None, q_ready=True, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    res = []
    for k in (0, 7, 0, 7):
        res.append((k, timed(k)))
    for m in mirrors:
        assert torch.equal(m, od[0])
    print(json.dumps({"mirrors_ms": [[k, round(t, 3)] for k, t in res]}))


if __name__ == "__main__":
    main()

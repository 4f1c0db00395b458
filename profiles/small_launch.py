"""Device time of one PPMM launch vs the number of moduli it carries (one
part, M = 2^14, K = 24576, N = 992): separates the per-launch overhead from
the per-modulus work. Optional env knobs (IRL_PPMM_CLUSTER ...) apply.

    python profiles/small_launch.py
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query
    from paper_2601_17561_b200.modmat import RnsBasis, Modulus, build_paper_basis
    full = build_paper_basis()
    N, M, K = 992, 1 << 14, 24576
    for nm in (1, 2, 3, 6, 24):
        b = RnsBasis()
        for md in full.moduli[:nm]:
            b.moduli.append(Modulus(md.p, md.e))
            b.Q *= md.p ** md.e
        eng = CcmmEngine(parts=1, m=M, k=K, max_n=N, basis=b)
        eng.synth_db(1)
        qd, _ = staging_tensors(eng, N)
        qd.copy_(torch.from_numpy(synth_query(2, K, N, eng.moduli).view(np.int16)))
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        eng.run_device(None, N, None, stream=s.cuda_stream)
        for _ in range(2):
            eng.run_device(None, N, None, q_ready=True, stream=s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(10):
            eng.run_device(None, N, None, q_ready=True, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(json.dumps({"moduli": nm, "ms_per_launch": ms, "ms_per_modulus": ms / nm}), flush=True)
        eng.close()


if __name__ == "__main__":
    main()

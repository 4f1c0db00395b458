"""Why is the e2e call slower than the device-resident step? Same process, c4
workload, alternating, medians: the device step alone; the step while an
unrelated 6.24 GB D2H (the step's output size) streams to pinned host memory
on another stream; the step while a 1.17 GB H2D streams in; and the e2e call.
Each run's SM clock and board power come from nvidia-smi.

    python profiles/e2e_interference.py [--reps 4]
"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--parts", type=int, default=8)
    a = ap.parse_args()
    import torch
    from bench import Clocks
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query
    N, M, K = 992, 1 << 14, 24576
    eng = CcmmEngine(parts=a.parts, m=M, k=K, max_n=N)
    eng.synth_db(1)
    qh = synth_query(2, K, N, eng.moduli)
    q = torch.from_numpy(qh.view(np.int16)).pin_memory()
    qn = q.numpy().view(np.uint16)
    out = torch.empty((a.parts, eng.nmod, N, M), dtype=torch.int16).pin_memory()
    outn = out.numpy().view(np.uint16)
    q_dev, out_dev = staging_tensors(eng, N)
    q_dev.copy_(q)
    junk_dev = torch.empty_like(out, device="cuda")
    junk_q = torch.empty_like(q, device="cuda")
    s = torch.cuda.Stream()
    side = torch.cuda.Stream()
    torch.cuda.synchronize()

    def step():
        eng.run_device(None, N, None, part0=0, nparts=0, q_ready=False, stream=s.cuda_stream)
        eng.run_device(None, N, None, part0=0, nparts=a.parts, q_ready=True, stream=s.cuda_stream)

    def d2h():
        with torch.cuda.stream(side):
            for i in range(a.parts):
                out[i].copy_(junk_dev[i], non_blocking=True)

    def h2d():
        with torch.cuda.stream(side):
            junk_q.copy_(q, non_blocking=True)

    variants = {
        "step": lambda: step(),
        "step+d2h": lambda: (d2h(), step()),
        "step+h2d": lambda: (h2d(), step()),
        "e2e": lambda: eng.run(qn, outn),
    }
    for fn in variants.values():
        fn()
        torch.cuda.synchronize()
    res = {k: [] for k in variants}
    for r in range(a.reps):
        order = list(variants) if r % 2 == 0 else list(reversed(variants))
        for kind in order:
            with Clocks(0) as clk:
                time.sleep(0.3)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                variants[kind]()
                e1.record(s)
                torch.cuda.synchronize()
                wall = (time.perf_counter() - t0) * 1e3
                gemm = e0.elapsed_time(e1)
            c = clk.summary()
            res[kind].append(wall)
            print(json.dumps({"rep": r, "kind": kind, "wall_ms": wall, "stream_ms": gemm, "sm_mhz": c["sm_mhz"],
                              "power_w": c["power_w_median"], "reasons": c["reasons"]}), flush=True)
    print(json.dumps({"summary": {k: statistics.median(v) for k, v in res.items()}}), flush=True)


if __name__ == "__main__":
    main()

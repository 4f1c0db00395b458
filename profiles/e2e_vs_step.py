"""Same-process A/B of the c4 device-resident step against the e2e call
(irl_ccmm_run, pinned host buffers), alternating, with the SM clock sampled
during each run. Attributes the e2e - step gap: clock (power) vs pipeline.

    python profiles/e2e_vs_step.py [--reps 6] [--parts 8] [--trace]

Prints one JSON line per run and a summary line.
"""
import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "profiles"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=6)
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
    out = torch.empty((a.parts, eng.nmod, N, M), dtype=torch.int16).pin_memory().numpy().view(np.uint16)
    q_dev, out_dev = staging_tensors(eng, N)
    q_dev.copy_(q)
    s = torch.cuda.Stream()
    torch.cuda.synchronize()

    def step():
        eng.run_device(None, N, None, part0=0, nparts=0, q_ready=False, stream=s.cuda_stream)
        eng.run_device(None, N, None, part0=0, nparts=a.parts, q_ready=True, stream=s.cuda_stream)

    def e2e():
        eng.run(qn, out)

    for _ in range(2):
        step()
        torch.cuda.synchronize()
        e2e()
    res = {"step": [], "e2e": []}
    for r in range(a.reps):
        for kind in ("step", "e2e") if r % 2 == 0 else ("e2e", "step"):
            with Clocks(0) as clk:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                if kind == "step":
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    step()
                    e1.record(s)
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1)
                else:
                    e2e()
                    ms = (time.perf_counter() - t0) * 1e3
            c = clk.summary()
            res[kind].append(ms)
            print(json.dumps({"rep": r, "kind": kind, "ms": ms, "sm_mhz": c["sm_mhz"],
                              "power_w": c["power_w_median"], "reasons": c["reasons"]}), flush=True)
    print(json.dumps({"summary": True, "parts": a.parts, "step_median_ms": statistics.median(res["step"]),
                      "e2e_median_ms": statistics.median(res["e2e"]),
                      "ratio": statistics.median(res["e2e"]) / statistics.median(res["step"])}), flush=True)


if __name__ == "__main__":
    main()

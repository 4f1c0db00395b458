"""Power / clock probe for the PPMM launch (energy budget under the 1 kW cap).

    python profiles/power_probe.py [--parts 4] [--secs 6]

Runs the CCMM PPMM back to back for --secs per variant while sampling
nvidia-smi (power, SM clock) and prints one JSON line per variant:
  * default            random DB + random query (the bench workload)
  * zero_db            DB digit planes all zero (tensor operands do not toggle)
  * zero_both          DB and query zero
  * cluster2           2-CTA clusters (no A multicast)
  * gate0              group gating off (more DRAM re-reads)
  * cl=PMxPN / gate=L  cluster shape / gate lead
The variants share one engine; knobs are the IRL_PPMM_* environment variables
read by the C ABI at each launch.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


class Smi:
    def __init__(self):
        self.lines = []

    def __enter__(self):
        self.p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,temperature.gpu",
                                   "--format=csv,noheader,nounits", "-lms", "100"],
                                  stdout=subprocess.PIPE, text=True)
        self.t = threading.Thread(target=lambda: [self.lines.append(x) for x in self.p.stdout], daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.p.terminate()
        self.p.wait()

    def summary(self):
        v = []
        for ln in self.lines:
            try:
                v.append([float(x) for x in ln.split(",")])
            except ValueError:
                pass
        v = v[len(v) // 4:]  # drop the ramp
        return {"sm_mhz": statistics.median(x[0] for x in v), "power_w": statistics.median(x[1] for x in v),
                "temp_c": max(x[2] for x in v), "samples": len(v)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", type=int, default=4)
    ap.add_argument("--rows", type=int, default=1 << 14)
    ap.add_argument("--k", type=int, default=24576)
    ap.add_argument("--n", type=int, default=992)
    ap.add_argument("--secs", type=float, default=6.0)
    ap.add_argument("--variants", default="default,cluster2,gate0,zero_db,zero_both")
    a = ap.parse_args()
    import torch
    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query

    eng = CcmmEngine(parts=a.parts, m=a.rows, k=a.k, max_n=a.n)
    eng.synth_db(1)
    q_dev, out_dev = staging_tensors(eng, a.n)
    q_rand = torch.from_numpy(synth_query(2, a.k, a.n, eng.moduli).view(np.int16))
    q_dev.copy_(q_rand)
    torch.cuda.synchronize()
    ops = 6.0 * eng.nmod * a.rows * a.n * a.k * a.parts

    def run(env, secs):
        for k in ("IRL_PPMM_CLUSTER", "IRL_PPMM_GATE"):
            os.environ.pop(k, None)
        os.environ.update(env)
        eng.run_device(None, a.n, None, q_ready=False)  # split + warm
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 0
        with Smi() as smi:
            t0 = time.time()
            e0.record()
            while time.time() - t0 < secs:
                eng.run_device(None, a.n, None, q_ready=True)
                n += 1
                if n % 4 == 0:
                    torch.cuda.synchronize()
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        r = smi.summary()
        r.update({"ms_per_launch": ms, "tops": ops / ms / 1e9,
                  "tops_per_ghz": ops / ms / 1e9 / (r["sm_mhz"] / 1e3),
                  "ops_per_joule_T": ops / 1e12 / (r["power_w"] * ms / 1e3)})
        return r

    ref_out = None
    zeroed = False
    for v in a.variants.split(","):
        if v == "zero_db":
            z = torch.zeros((eng.nmod, a.rows, a.k), dtype=torch.int16, device="cuda")
            for g in range(a.parts):
                eng.load_part(g, z)
            del z
            zeroed = True
            torch.cuda.synchronize()
            r = run({}, a.secs)
        elif v.startswith("db_"):
            # DB digit distribution experiments: residues v = d0 + p d1 (mod p^2)
            # with both centred digits drawn from a sub-range (energy vs data)
            kind = v[3:]
            g = torch.Generator(device="cuda").manual_seed(5)
            res = torch.empty((eng.nmod, a.rows, a.k), dtype=torch.int16, device="cuda")
            for i, (pp, ee) in enumerate(zip(eng.primes, eng.exps)):
                pp = int(pp)
                h = (pp - 1) // 2
                lo, hi = {"pos": (0, h), "neg": (-h, 0), "small": (-(h // 2), h // 2),
                          "full": (-h, h), "tiny": (-3, 3)}[kind]
                d0 = torch.randint(lo, hi + 1, (a.rows, a.k), generator=g, device="cuda", dtype=torch.int32)
                d1 = torch.randint(lo, hi + 1, (a.rows, a.k), generator=g, device="cuda", dtype=torch.int32)
                res[i] = ((d0 + pp * d1) % (pp * pp)).to(torch.int16)
            for gi in range(a.parts):
                eng.load_part(gi, res)
            del res
            zeroed = True
            torch.cuda.synchronize()
            r = run({}, a.secs)
        elif v == "zero_both":
            q_dev.zero_()
            r = run({}, a.secs)
            q_dev.copy_(q_rand)
            torch.cuda.synchronize()
        elif v == "cluster2":
            r = run({"IRL_PPMM_CLUSTER": "2"}, a.secs)
        elif v == "gate0":
            r = run({"IRL_PPMM_GATE": "0"}, a.secs)
        elif v.startswith("cl="):
            r = run({"IRL_PPMM_CLUSTER": v[3:]}, a.secs)
        elif v.startswith("gate="):
            r = run({"IRL_PPMM_GATE": v[5:]}, a.secs)
        else:
            r = run({}, a.secs)
        r["variant"] = v
        if not zeroed and not v.startswith("zero"):
            # every schedule / cluster shape must produce the identical output
            if ref_out is None:
                ref_out = out_dev.clone()
            else:
                r["same_output"] = bool(torch.equal(ref_out, out_dev))
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()

"""Measured int8 tensor peak on this box: cuBLASLt int8 GEMM (torch._int_mm,
int8 x int8 -> int32) at 8192^3 and 16384 x 16384 x 8192, operands uniform
in [-125, 125] like the PPMM digits. Burst = best of 10; sustained = back to
back for --secs seconds (the power-capped figure a 150 ms kernel sees), with
nvidia-smi clocks sampled during the sustained run.

    python profiles/int8_peak.py [--secs 6]
"""
import argparse
import json
import statistics
import subprocess
import threading
import time


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--secs", type=float, default=6.0)
    a = ap.parse_args()
    import torch
    out = {}
    for (m, n, k) in ((8192, 8192, 8192), (16384, 16384, 8192)):
        A = torch.randint(-125, 126, (m, k), dtype=torch.int8, device="cuda")
        B = torch.randint(-125, 126, (n, k), dtype=torch.int8, device="cuda").t()  # column-major K x N
        for _ in range(3):
            torch._int_mm(A, B)
        torch.cuda.synchronize()
        ops = 2.0 * m * n * k
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(A, B)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        lines = []
        p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw",
                              "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)
        th = threading.Thread(target=lambda: [lines.append(x) for x in p.stdout], daemon=True)
        th.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cnt = 0
        t0 = time.time()
        e0.record()
        while time.time() - t0 < a.secs:
            for _ in range(8):
                torch._int_mm(A, B)
            cnt += 8
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        p.terminate()
        sus = e0.elapsed_time(e1) / cnt
        v = []
        for ln in lines:
            try:
                v.append([float(x) for x in ln.split(",")])
            except ValueError:
                pass
        v = v[len(v) // 3:]
        out[f"{m}x{n}x{k}"] = {"burst_tops": ops / best / 1e9, "sustained_tops": ops / sus / 1e9,
                               "sm_mhz": statistics.median(x[0] for x in v) if v else None,
                               "power_w": statistics.median(x[1] for x in v) if v else None}
        print(json.dumps({f"{m}x{n}x{k}": out[f"{m}x{n}x{k}"]}), flush=True)


if __name__ == "__main__":
    main()

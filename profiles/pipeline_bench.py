"""The reference's own Alg. 1 + Alg. 2 pipeline (acceptance.cpp full_config:
n_db 4096, d 1024, rho 31, batch 4; run_instances from seed 60000), timed per
instance with the stock Emulator::ccmm_twin and with its product from the B200
engine (oracle/_ref/libirl_pipe_{ref,b200}.so). The results
of both must be identical; the time difference is the CCMM's share.

    python profiles/pipeline_bench.py [--instances 3]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", type=int, default=3)
    a = ap.parse_args()
    import oracle_lib as ol
    fc = np.ascontiguousarray(ol.FOLD_POLY_APPC, np.float64)
    res = {}
    for kind in ("b200", "ref", "b200"):
        lib = ol.pipe(kind)
        lib.irl_hook_reset()
        out = np.zeros((a.instances, 2, 16), np.int64)
        t0 = time.perf_counter()
        st = lib.pipe_instances(31, 4, 4096, a.instances, 60000, fc.ctypes.data_as(ol.C.POINTER(ol.C.c_double)),
                                len(fc), ol.ptr(out, ol.i64p), 16)
        secs = time.perf_counter() - t0
        assert st == 0, lib.pipe_last_error()
        res[kind] = (out, lib.irl_hook_digest())
        print(json.dumps({"ccmm_twin": kind, "instances": a.instances, "s_per_instance": secs / a.instances,
                          "agree_all": bool(out[:, :, 0].all()), "digest": hex(lib.irl_hook_digest())}), flush=True)
    print(json.dumps({"identical": bool((res["ref"][0] == res["b200"][0]).all()) and res["ref"][1] == res["b200"][1]}))


if __name__ == "__main__":
    main()

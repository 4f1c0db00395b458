"""Benchmark of the RGSW CCMM hot path on B200 (BASELINE.json north star).

Workload (BASELINE.json configs[3] at N GPUs; configs[1-2] are its per-slice
pieces): a 32-eye x 31-rotation query batch (N = 992 columns) against the full
database of 7 * 2^14 templates in the paper's 8-part layout (shared a-part +
7 b-part slices of 2^14 rows), K = d2 + N_qry = 2^14 + 2^13 = 24576, modulus
Q = prod_{127<=p<=253} p^2 (24 primes, 361 bits). One step = split the query
into digit planes + 8 K-concatenated PPMMs mod Q (4 RGSW PPMMs per a/b pair)
+ the a-part result broadcast (N > 1). Inputs are synthetic residues from the
counter generator (uniform mod p^2), DB planes resident in HBM (144 GiB at
N = 1, far above L2, so no flush is needed between steps).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from types import SimpleNamespace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = ("CCMM latency per 32×31 query batch vs 7·2^14 DB; int8 TOPS and % of tensor peak")
UNIT = "int8 TOPS (6*P*M*N*K per part, unpadded)"
DATASHEET_INT8_TOPS = 4500.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--parts", type=int, default=8)
    ap.add_argument("--rows", type=int, default=1 << 14, help="templates per part (M; the a-part's rows)")
    ap.add_argument("--b-rows", type=int, default=0,
                    help="templates per b-part (default --rows; c5 grows them to 2^17)")
    ap.add_argument("--deal", choices=["auto", "parts", "blocks"], default="auto",
                    help="multi-GPU dealing: whole parts, or balanced row blocks (dist.deal_blocks; auto = blocks "
                         "when b-parts are taller than the a-part)")
    ap.add_argument("--k", type=int, default=(1 << 14) + (1 << 13), help="d2 + N_qry")
    ap.add_argument("--eyes", type=int, default=32)
    ap.add_argument("--rot", type=int, default=31)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=32, help="DB rows per (part, modulus) task in the CPU sample")
    ap.add_argument("--no-int8-ref", action="store_true", help="skip the live cuBLASLt int8 comparison")
    ap.add_argument("--exchange", choices=["auto", "mirror", "broadcast"], default="auto",
                    help="a-part exchange at N>1: fused P2P epilogue stores (mirror, validated in warm-up, "
                         "falls back to broadcast) or the NCCL broadcast")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo + --same-device: run the multi-rank paths with every rank on one GPU (tests)")
    ap.add_argument("--same-device", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--e2e-query", choices=["auto", "host"], default="auto",
                    help="N>1 e2e: auto shards the query H2D over ranks + all-gather when H2D-bound")
    ap.add_argument("--moddown", type=int, default=0, metavar="DROP",
                    help="f2 in the step: ModDown every local output to Q/Delta (drop the last DROP moduli) "
                         "and exchange the rescaled a-part (NCCL broadcast of (24-DROP)/24 of the bytes)")
    ap.add_argument("--config", choices=["c2", "c3", "c4"], default="c4",
                    help="BASELINE.json config: c2 one DB slice as one PPMM (K = 2^14), c3 a-part + one "
                         "b-part, c4 the full 8-part DB (default; the headline metric)")
    a = ap.parse_args()
    a.b_rows = a.b_rows or a.rows
    if a.config == "c2":
        a.parts, a.k = 1, 1 << 14
    elif a.config == "c3":
        a.parts = 2
    return a


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            try:
                pw.append(float(f[3]))
            except ValueError:
                pass
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(pw) if pw else None}


# ---------------------------------------------------------------------------
# CPU reference leg (oracle/_ref = unmodified reference modmat.cpp; else the port)
# ---------------------------------------------------------------------------

def host_cpu():
    """Host CPU model and the threads this process may use (lscpu)."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:  # noqa: BLE001
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        usable = os.cpu_count() or 1
    return {"model": model, "threads_usable": usable, "cpu_count": os.cpu_count()}


def loaded_repo_libs():
    """Shared objects under this repo mapped into the process (evidence of
    which native code ran)."""
    libs = set()
    try:
        for ln in open("/proc/self/maps"):
            f = ln.split()
            if len(f) >= 6 and f[-1].endswith(".so") and str(ROOT) in os.path.realpath(f[-1]):
                libs.add(os.path.relpath(os.path.realpath(f[-1]), os.path.realpath(ROOT)))
    except OSError:
        pass
    return sorted(libs)


def query_residues_oracle(K, N, moduli):
    """The step's query residues [nmod][K][N] from the oracle's copy of the
    counter generator (seed 2, stream 0xFF; identical to ccmm.synth_query), so
    the reference arm never loads the product library."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as ol
    return np.stack([ol.synth_block(2, 0xFF, i, 0, K, 0, N, m) for i, m in enumerate(moduli)])


def cpu_reference_sample(args, moduli, q_host, rows=None, threads=None, parts=None):
    """Times the reference gemm_mod_psq (modmat.cpp:143-160) on a bounded sample
    of the same workload: `rows` DB rows x full K x all N query columns, for
    every modulus of parts `parts` (one task per (part, modulus)); tasks spread
    over host threads (the function is pure). Test
    infrastructure only (tests/oracle_lib.py -> oracle/_ref, else the port)."""
    import ctypes as C
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as ol

    rows = rows or args.cpu_rows
    threads = threads or host_cpu()["threads_usable"]
    parts = tuple(parts) if parts is not None else tuple(range(args.parts))
    K, N = args.k, args.eyes * args.rot
    kind = "reference" if ol.ref_available() else "port"
    A, B, Cc, P = [], [], [], []
    for part in parts:
        for i, m in enumerate(moduli):
            A.append(np.ascontiguousarray(ol.synth_block(args.seed, part, i, 0, rows, 0, K, m).astype(np.int32)))
            B.append(np.ascontiguousarray(q_host[i].astype(np.int32)))
            Cc.append(np.zeros((rows, N), np.int32))
            P.append(int(round(m ** 0.5)))
    ntasks = len(A)
    t0 = time.perf_counter()
    if kind == "reference":
        lib = ol.ref()
        arr = lambda xs: (ol.i32p * len(xs))(*[x.ctypes.data_as(ol.i32p) for x in xs])  # noqa: E731
        st = lib.ref_gemm_mod_psq_batch(arr(A), arr(B), arr(Cc), (C.c_uint32 * ntasks)(*P), ntasks, rows, K, N,
                                        threads)
        assert st == 0, lib.ref_last_error()
    else:
        from concurrent.futures import ThreadPoolExecutor

        def task(j):
            st, c = ol.orc_gemm_mod_psq(A[j], B[j], P[j])
            assert st == 0
            Cc[j][...] = c
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(task, range(ntasks)))
    secs = time.perf_counter() - t0
    ops = 6.0 * rows * N * K * ntasks
    return {"kind": kind, "seconds": secs, "ops": ops, "tops": ops / secs / 1e12, "threads": threads,
            "rows": rows, "tasks": ntasks, "outputs": Cc, "parts": parts,
            "sample": (f"{rows} DB rows x K={K} x N={N} for each of {len(moduli)} moduli of parts "
                       f"{list(parts)} ({ntasks} gemm_mod_psq calls, {kind} code, {threads} threads); "
                       f"rate extrapolated linearly in M (cost ~ M*N*K)")}


def run_reference_arm(args):
    """The reference's own CPU implementation (oracle/_ref: unmodified
    modmat.cpp gemm_mod_psq) on the box's host cores, same metric/config. Loads
    only oracle/ libraries (never the product package). Each step samples
    args.cpu_rows DB rows of two parts (rotating over the 8) x every modulus."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as ol
    pr, ex = ol.paper_basis()
    moduli = [int(p) ** int(e) for p, e in zip(pr, ex)]
    N = args.eyes * args.rot
    total_ops = 6.0 * len(moduli) * total_rows(args) * N * args.k
    q = query_residues_oracle(args.k, N, moduli)
    rates, secs = [], []
    last = None
    for it in range(args.warmup + args.steps):
        parts = [(2 * it + j) % args.parts for j in range(min(2, args.parts))]
        r = cpu_reference_sample(args, moduli, q, parts=parts)
        if it >= args.warmup:
            rates.append(r["tops"])
            secs.append(r["seconds"])
        last = r
    v = statistics.median(rates)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": statistics.mean(secs) * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32 (int8 digits)", "data": "synthetic",
            "impl": "reference",
            "config": config_dict(args, len(moduli)),
            "step_definition": "one bounded CPU sample (see cpu_baseline.sample); ms_per_step is its measured time",
            "ccmm_latency_ms_extrapolated": total_ops / (v * 1e12) * 1e3,
            "host_cpu": host_cpu(),
            "loaded_repo_libs": loaded_repo_libs(),
            "product_package_imported": "paper_2601_17561_b200" in sys.modules,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": last["threads"], "kind": last["kind"],
                             "sample": last["sample"].replace(f"parts {list(last['parts'])}",
                                                              "2 parts per step (rotating over all)")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def nccl_summary(path, world):
    """What NCCL_DEBUG=INFO recorded about the communicator (rank 0's file)."""
    if not path or world < 2:
        return None
    try:
        lines = Path(path).read_text(errors="replace").splitlines()
    except OSError:
        return {"debug_file": path, "read": False}
    init = [ln for ln in lines if "Init COMPLETE" in ln]
    return {"debug_file": path, "lines": len(lines), "init_complete": init[:1],
            "nranks_seen": sorted({int(t.split()[1]) for ln in init for t in [ln[ln.find("nranks"):]]
                                   if t.startswith("nranks ") and t.split()[1].isdigit()}),
            "nvls": any("NVLS" in ln and "enabled" in ln.lower() for ln in lines) or
                    any("NVLS multicast support is available" in ln for ln in lines),
            "version": next((ln.split("NCCL version", 1)[1].strip() for ln in lines if "NCCL version" in ln), None)}


WORKLOADS = {
    "c2": "c2: full-RNS PPMM mod Q on one DB slice, 992 query columns x d = 2^14 x 2^14 templates",
    "c3": "c3: RGSW CCMM a-part + one b-part (2 K-concatenated PPMMs, N_db = 2^14, K = 2^14 + 2^13)",
    "c4": "c4: 32x31 query batch vs full DB 7*2^14 templates, 8-part RGSW layout (a-part + 7 b-parts)",
}


def total_rows(args):
    """Database rows over all parts: the a-part plus parts - 1 b-parts."""
    return args.rows + (args.parts - 1) * args.b_rows


def config_dict(args, nmod):
    N = args.eyes * args.rot
    extra = {}
    if args.moddown:
        extra = {"moddown_drop": args.moddown,
                 "moddown": f"every local output rescaled to Q/Delta (last {args.moddown} moduli dropped) inside "
                            "the step; the a-part exchange carries the rescaled result"}
    return {"workload": WORKLOADS[args.config] + (" + ModDown" if args.moddown else ""), **extra,
            "parts": args.parts, "templates_per_part": args.rows,
            **({"templates_per_b_part": args.b_rows} if args.b_rows != args.rows else {}),
            "K": args.k, "query_columns": N,
            "eyes": args.eyes, "rotations": args.rot, "moduli": nmod, "log2_Q": 360.8156,
            "digit_planes": 2 * nmod, "parallelism": f"db-slices over {args.gpus} GPU(s)",
            "l2": "inputs larger than L2 (DB digit planes, 18 GiB per part)"}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def measure_split(R):
    """The query split kernel alone (HBM-bound): 10 back-to-back launches."""
    torch, eng, N, K, nmod, stream, hbm_peak = R.torch, R.eng, R.N, R.K, R.nmod, R.stream, R.hbm_peak
    # ---- the query split (HBM-bound): 2 B read + 2 B written per (entry, modulus)
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    eng.run_device(None, N, None, part0=0, nparts=0, q_ready=False, stream=stream.cuda_stream)
    s0.record(stream)
    for _ in range(10):
        eng.run_device(None, N, None, part0=0, nparts=0, q_ready=False, stream=stream.cuda_stream)
    s1.record(stream)
    torch.cuda.synchronize()
    split_ms = s0.elapsed_time(s1) / 10
    split_bytes = 4.0 * nmod * K * N
    split_roof = {"bound": "hbm", "kernel": "split_cols_u16_vec_kernel", "launch_ms": split_ms,
                  "achieved": split_bytes / (split_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                  "frac": split_bytes / (split_ms * 1e-3) / 1e9 / hbm_peak, "bytes_per_launch": split_bytes,
                  "note": "10 back-to-back query splits, CUDA events; input and output (1.17 GB each) "
                          "exceed L2"}
    return split_roof


def measure_ingest(R):
    """The mod-Q ingest kernel (f3: 46-byte BigMatrix entries -> residues ->
    digit planes, irl_split_bigint) on 2048 x K device-resident entries, 5
    launches, CUDA events: 46 B read + 48 B written per entry. Not part of the
    step (a database is ingested once)."""
    import ctypes as C
    torch, ctx, K, hbm_peak, rank = R.torch, R.ctx, R.K, R.hbm_peak, R.rank
    if rank != 0:
        return None
    from paper_2601_17561_b200 import capi
    from paper_2601_17561_b200.modmat import build_paper_basis
    b = build_paper_basis()
    p, e = b.arrays()
    w, rows = b.width(), 2048
    g = torch.Generator(device="cuda").manual_seed(7)
    ent = torch.randint(0, 256, (rows * K, w), dtype=torch.uint8, device="cuda", generator=g)
    ent[:, -1] = 0  # below 2^360 < Q
    ldk = (K + 15) // 16 * 16
    planes = torch.empty((len(p), 2, rows, ldk), dtype=torch.int8, device="cuda")
    s = torch.cuda.current_stream()

    def run():
        ctx.check(capi.lib().irl_split_bigint(ctx.handle, C.c_void_p(ent.data_ptr()), w, rows, K, 0,
                                               capi.ptr(p, capi.u32p), capi.ptr(e, capi.u32p), len(p),
                                               C.c_void_p(planes.data_ptr()), ldk, C.c_void_p(s.cuda_stream)))
    run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(5):
        run()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    nbytes = rows * K * (w + 2 * len(p))
    del ent, planes
    return {"bound": "hbm", "kernel": "split_bigint_words_kernel", "launch_ms": ms,
            "achieved": nbytes / (ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": nbytes / (ms * 1e-3) / 1e9 / hbm_peak, "bytes_per_launch": nbytes,
            "entries_per_s": rows * K / (ms * 1e-3),
            "note": "not part of the CCMM step: f3 ingest of 46-byte mod-Q entries into digit planes "
                    "(integer-multiply bound; the file reads that feed it run at ~13-15 GB/s)"}


def measure_moddown(R):
    """f2 ModDown of all local outputs (HBM-bound), outside the step."""
    torch, eng, N, M, nmod, stream, local_parts = R.torch, R.eng, R.N, R.M, R.nmod, R.stream, R.local_parts
    hbm_peak = R.hbm_peak
    # ---- ModDown of the step's outputs (f2; HBM-bound): drop the last 3 moduli
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    drop = 3
    md_dst = torch.empty((1, nmod - drop, N, M), dtype=torch.int16, device="cuda")
    for p_ in range(local_parts.count):
        eng.rescale(N, md_dst, drop, True, part0=p_, nparts=1, stream=stream.cuda_stream)
    s0.record(stream)
    for p_ in range(local_parts.count):
        eng.rescale(N, md_dst, drop, True, part0=p_, nparts=1, stream=stream.cuda_stream)
    s1.record(stream)
    torch.cuda.synchronize()
    md_ms = s0.elapsed_time(s1)
    md_bytes = 2.0 * (2 * nmod - drop) * N * M * local_parts.count
    moddown = {"bound": "hbm", "kernel": "rescale_kernel", "drop_moduli": drop, "ms_per_step": md_ms,
               "achieved": md_bytes / (md_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
               "frac": md_bytes / (md_ms * 1e-3) / 1e9 / hbm_peak, "bytes": md_bytes,
               "note": "not part of the CCMM step: f2 rescale of all local outputs to Q/Delta, "
                       "Delta = product of the last 3 moduli (~2^47)"}
    del md_dst
    return moddown


def measure_e2e(R):
    """The same step end to end through the public C ABI with host buffers."""
    args, torch, dist, eng, N, M, K, nmod, world = R.args, R.torch, R.dist, R.eng, R.N, R.M, R.K, R.nmod, R.world
    rank, local_parts, out_dev, q_dev, q_pinned = R.rank, R.local_parts, R.out_dev, R.q_dev, R.q_pinned
    q_host, a_out, exchange, md_drop, out_md, total_ops = R.q_host, R.a_out, R.exchange, R.md_drop, R.out_md, R.total_ops
    # ---- end to end through the public C ABI with host buffers -------------
    e2e = None
    if not args.no_e2e:
        out_host = torch.empty((local_parts.count, nmod, N, M), dtype=torch.int16).pin_memory()
        q_np = q_pinned.numpy().view(np.uint16)
        o_np = out_host.numpy().view(np.uint16)
        # H2D-bound layouts (few parts per GPU: GEMM time per modulus below its
        # H2D time, the engine's own planner criterion) distribute the query
        # over NVLink instead: each rank copies 1/N of the moduli from the host
        # and all-gathers the rest, then runs split + GEMM + part-granular D2H
        # (irl_ccmm_run_dq). Otherwise irl_ccmm_run pipelines the full H2D.
        sharded = (world > 1 and local_parts.count * M < 20000 and nmod % world == 0
                   and args.e2e_query != "host")
        per = nmod // world if sharded else nmod
        lo = rank * per if sharded else 0
        q_bytes = q_dev.view(torch.uint8)  # [nmod][K][2N]: gloo and NCCL both carry uint8
        q_slices = [q_bytes[r_ * per:(r_ + 1) * per] for r_ in range(world)] if sharded else None

        q_events = []

        def e2e_once():
            R.next_slot()
            if sharded:
                cs = torch.cuda.current_stream()
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record(cs)
                q_dev[lo:lo + per].copy_(q_pinned.view(nmod, K, N)[lo:lo + per], non_blocking=True)
                dist.all_gather(q_slices, q_bytes[lo:lo + per].clone() if args.backend == "gloo" else q_bytes[lo:lo + per])
                ev[1].record(cs)
                q_events.append(ev)
                eng.run_dq(None, N, o_np, stream=cs.cuda_stream)
            else:
                eng.run(q_np, o_np)  # H2D query, split, all local PPMMs, D2H outputs
            if md_drop:  # the engine's device outputs of the run, rescaled for the exchange
                eng.rescale(N, out_md, md_drop, True, stream=torch.cuda.current_stream().cuda_stream)
            if world > 1:
                # the a-part result exchange stays on the device
                if exchange == "mirror":  # the owner's epilogue already stored out_A into the peers
                    w = dist.all_reduce(torch.zeros(1, dtype=torch.int32, device="cuda"), async_op=True)
                else:
                    w = dist.broadcast(a_out().view(torch.uint8), src=0, async_op=True)
                w.wait()
                torch.cuda.synchronize()

        if world > 1:
            dist.barrier()
        for _ in range(max(1, args.warmup - 1)):
            e2e_once()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        q_events.clear()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_once()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        per_rank_e2e = None
        if world > 1:  # this rank's e2e and, when sharded, its query H2D + all-gather time
            mine = {"rank": rank, "e2e_ms": e2e_ms,
                    "query_in_ms": statistics.mean(a.elapsed_time(b) for a, b in q_events) if q_events else None}
            per_rank_e2e = [None] * world
            dist.all_gather_object(per_rank_e2e, mine)
        # the e2e outputs (host) must equal the device-resident step's (same
        # query): a 64-row block of every part and modulus, on every rank
        cols = min(M, 64)
        same = bool((out_dev[:, :, :, :cols].cpu().numpy().view(np.uint16) == o_np[:, :, :, :cols]).all())
        ok_t = torch.tensor([1 if same else 0], dtype=torch.int32, device="cuda")
        if world > 1:
            dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
        e2e_exact = bool(ok_t.item())
        tt = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
        e2e = {"value": total_ops / (e2e_ms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(q_host.nbytes // world if sharded else q_host.nbytes),
               "d2h_bytes_per_step": int(local_parts.count * nmod * N * M * 2),
               "outputs_equal_device_step": e2e_exact, "per_rank": per_rank_e2e,
               "call": (f"1/N of the query H2D per rank + {args.backend.upper()} all-gather, then irl_ccmm_run_dq "
                        "(include/irl_capi.h) with pinned host outputs") if sharded else
                       "irl_ccmm_run (include/irl_capi.h) with pinned host buffers"}
    return e2e


def measure_dist_check(R):
    """N > 1: sampled rows of every rank against the CPU oracle; a-part consistency."""
    args, torch, dist, M, K, nmod, world, local_parts = R.args, R.torch, R.dist, R.M, R.K, R.nmod, R.world, R.local_parts
    out_dev, q_host, moduli, a_out = R.out_dev, R.q_host, R.moduli, R.a_out
    # ---- N > 1: every rank checks sampled rows of its first local part against
    # the CPU oracle (test infrastructure, oracle/irl_oracle.c), folded with MIN
    dist_check = None
    if world > 1 and not args.no_cpu_baseline:
        sys.path.insert(0, str(ROOT / "tests"))
        import oracle_lib as ol
        part_g, row0 = R.unit_map[0]  # global part and first row of the first local unit
        rows = np.array([0, M // 2, M - 1], np.uint32)
        got_all = out_dev[0].cpu().numpy().view(np.uint16)  # [nmod][N][M] of the first local unit
        ok = True
        for i, m_ in enumerate(moduli):
            qt = np.ascontiguousarray(q_host[i].T)
            for r_ in rows:  # only the sampled DB rows are generated
                a_row = ol.synth_block(args.seed, part_g, i, row0 + int(r_), 1, 0, K, m_)
                want = ol.ppmm_rows_direct(a_row, qt, np.zeros(1, np.uint32), m_)
                ok &= bool((got_all[i][:, int(r_)] == want[0]).all())
        ok_t = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
        dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
        dist_check = {"rows_per_rank": int(len(rows)), "moduli": nmod, "bit_exact_all_ranks": bool(ok_t.item()),
                      "oracle": "oracle/irl_oracle.c (pinned to the reference)"}
        # every rank holds the same a-part result after the exchange
        a_sum = torch.sum(a_out().to(torch.int64)).view(1)
        sums = [torch.zeros_like(a_sum) for _ in range(world)]
        dist.all_gather(sums, a_sum)
        dist_check["a_part_identical_all_ranks"] = len({int(x.item()) for x in sums}) == 1
    return dist_check


def measure_cpu(R):
    """The CPU baseline (rank 0, N = 1) with a bit-exact check of its rows."""
    args, nmod, world, rank, out_dev, q_host = R.args, R.nmod, R.world, R.rank, R.out_dev, R.q_host
    moduli, total_ops = R.moduli, R.total_ops
    # ---- CPU baseline (rank 0, N = 1) with a bit-exact check of its rows ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference_sample(args, moduli, q_host=q_host)
        gpu_rows = out_dev[:, :, :, : r["rows"]].cpu().numpy().view(np.uint16)
        exact = True
        j = 0
        for part in r["parts"]:
            unit = R.unit_map.index((part, 0))  # rows [0, cpu_rows) of global part `part`
            for i in range(nmod):
                exact &= bool((r["outputs"][j] == gpu_rows[unit, i].T).all())
                j += 1
        cpu = {"value": r["tops"], "unit": UNIT, "cores": r["threads"], "kind": r["kind"],
               "sample": r["sample"], "seconds": r["seconds"], "bit_exact_vs_gpu": exact,
               "bit_exact_parts": list(r["parts"]), "bit_exact_rows_per_part": r["rows"],
               "host_cpu": host_cpu(),
               "extrapolated_ccmm_latency_s": total_ops / (r["tops"] * 1e12)}
    return cpu


def stand_in_fold_chain():
    """Three classifier stages of degrees 15, 31 and 3 (smooth sign approximants,
    composed): the reference designs its chains offline (compose_classifier,
    poly_design.cpp); the evaluation cost depends only on the degrees."""
    from numpy.polynomial import polynomial as P

    def compose(p, q):
        out = np.array([0.0])
        for c in p[::-1]:
            out = P.polyadd(P.polymul(out, q), [c])
        return out
    f3 = np.array([0.0, 1.5, 0.0, -0.5])
    f5 = np.array([0.0, 15, 0, -10, 0, 3]) / 8.0
    f15 = compose(f3, f5) * (1 / 1024.0) ** np.arange(16)
    f31 = np.r_[compose(f3, compose(f3, f3)), 0.0, 0.0, 0.0, 1e-9]
    return [(0.365, f15), (0.0, f31), (0.0, np.array([0.5, 0.75, 0.0, -0.25]))]


def measure_fold(R):
    """The next stage after the CCMM (f4, csrc/fold.cu): Alg. 2's fold stage on
    this step's geometry -- the query columns against the b-part templates
    (blocks of d = 2^14), fold_k = 16 -- on device-resident products and
    overlaps, 10 launches, CUDA events. 8 B read per (column, template) + 8 B
    written per output slot; the inputs (0.9 GB at c4) exceed L2."""
    args, torch, N, M, rank, hbm_peak = R.args, R.torch, R.N, R.M, R.rank, R.hbm_peak
    if rank != 0 or args.rot < 1:
        return None
    from paper_2601_17561_b200.fold import FoldConfig, fold_stage_device
    d = 1 << 14
    n_db = max(1, (args.parts - 1) * args.b_rows // d) * d  # the b-part templates, whole blocks
    eyes, rho, fold_k = args.eyes, args.rot, min(16, args.rot)
    g = torch.Generator(device="cuda").manual_seed(3)
    ovl = torch.randint(1, d, (N, n_db), dtype=torch.int32, device="cuda", generator=g)
    inner = (torch.rand((N, n_db), device="cuda", generator=g) * (2 * ovl + 1)).to(torch.int32) - ovl
    refolded = torch.empty(eyes * (n_db // d) * d, dtype=torch.float64, device="cuda")
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    cfg = FoldConfig(rho=rho, fold_k=fold_k, d=d, fold_chain=stand_in_fold_chain(), negative=(-0.05, 0.05))
    s = torch.cuda.current_stream()
    for _ in range(3):
        fold_stage_device(inner, ovl, eyes, cfg, None, refolded, flags, stream=s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        fold_stage_device(inner, ovl, eyes, cfg, None, refolded, flags, stream=s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    nbytes = 8.0 * N * n_db + 8.0 * refolded.numel()
    del inner, ovl, refolded
    return {"bound": "hbm", "kernel": "fold_stage_kernel", "launch_ms": ms,
            "achieved": nbytes / (ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": nbytes / (ms * 1e-3) / 1e9 / hbm_peak, "bytes_per_launch": nbytes,
            "pairs": N * n_db,
            "note": f"not part of the CCMM step: Alg. 2 fold stage (normalize, degree-7 fold polynomial with "
                    f"Rot alignment, 3-stage fold chain, refold) on {N} columns x {n_db} templates, fold_k "
                    f"{fold_k}; exact IEEE double, FP64/issue-bound (DESIGN.md 3)"}


def measure_iris(R):
    """The plaintext scoring stage on the same query geometry (f4, csrc/iris.cu):
    a registered database of the 7 * 2^14 b-part templates (d = 2^14), the
    eyes x rotations batch, match bits out; the ternary / mask products run on
    the block-scaled FP4 tensor path, the query columns on M (one pass over the
    database). Host wall clock per call (query bits in, match bits out into a
    reused pinned buffer), median of 10."""
    args, rank, M = R.args, R.rank, R.M
    if rank != 0:
        return None
    import os as _os

    from paper_2601_17561_b200.iris import IrisDatabase, Interval
    d = 1 << 14
    n_db = max(1, (args.parts - 1) * args.b_rows // d) * d
    eyes, rho = args.eyes, args.rot
    rng = np.random.default_rng(5)
    words = d // 64
    bits = lambda n: rng.integers(0, 1 << 63, size=(n, words), dtype=np.uint64)  # noqa: E731
    dc, dm, qc, qm = bits(n_db), bits(n_db) | bits(n_db), bits(eyes), bits(eyes) | bits(eyes)
    db = IrisDatabase.from_packed(dc, dm, d, eyes * rho)
    # one caller-owned, page-locked output buffer reused per batch (as the CCMM
    # e2e uses pinned host buffers): the match bits are DMA'd straight into it
    out_bits = R.torch.zeros((eyes, n_db), dtype=R.torch.uint8).pin_memory().numpy()
    try:
        for _ in range(3):
            db.match_packed(qc, qm, eyes, rho, Interval(0.35, 1.0), out_bits=out_bits)
        ts = []
        for _ in range(10):
            t0 = time.perf_counter()
            db.match_packed(qc, qm, eyes, rho, Interval(0.35, 1.0), out_bits=out_bits)
            ts.append((time.perf_counter() - t0) * 1e3)
    finally:
        db.close()
    ms = statistics.median(ts)
    ops = 4.0 * n_db * eyes * rho * d  # two products, 2 ops per multiply-add
    return {"stage": "irl_iris_db_match (registered database, host buffers: query bits in, "
                     "match bits out into a reused pinned buffer)", "ms": ms,
            "effective_tops": ops / (ms * 1e-3) / 1e12, "n_db": n_db, "columns": eyes * rho, "d": d,
            "tensor_path": "int8 (IRL_IRIS_I8)" if _os.environ.get("IRL_IRIS_I8") else
                           "FP4 e2m1, tcgen05 kind::mxf4.block_scale, unit scales, FP32 accumulate (exact)",
            "note": "not part of the CCMM step"}


def measure_int8(R):
    """Live library comparison: cuBLASLt int8 GEMM on this box."""
    args, torch, rank = R.args, R.torch, R.rank
    # ---- live library comparison: cuBLASLt int8 GEMM (torch._int_mm) on this box,
    # same operand distribution, back to back for 3 s after the timed region
    int8_ref = None
    if rank == 0 and not args.no_int8_ref:
        torch.cuda.set_stream(torch.cuda.default_stream())
        A8 = torch.randint(-125, 126, (8192, 8192), dtype=torch.int8, device="cuda")
        B8 = torch.randint(-125, 126, (8192, 8192), dtype=torch.int8, device="cuda").t()
        for _ in range(3):
            torch._int_mm(A8, B8)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        cnt, t0 = 0, time.time()
        e0.record()
        while time.time() - t0 < 3.0:
            for _ in range(8):
                torch._int_mm(A8, B8)
            cnt += 8
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        int8_ref = {"library": "cuBLASLt int8 GEMM via torch._int_mm, 8192^3, operands uniform in [-125, 125]",
                    "sustained_tops": 2.0 * 8192 ** 3 / (e0.elapsed_time(e1) / cnt) / 1e9,
                    "note": "a plain int8 GEMM (1 product); the PPMM does 3 fused products + mod-p^2 epilogue"}
        del A8, B8
    return int8_ref


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_device:
        local = 0  # test harness: every rank on GPU 0 (multi-rank code paths on a 1-GPU box)
    torch.cuda.set_device(local)
    nccl_log = None
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.backend == "nccl":
            # NCCL's own record of the communicator (ranks, channels, NVLS),
            # to a per-rank file so stdout keeps the one JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            nccl_log = os.environ.setdefault("NCCL_DEBUG_FILE", f"/tmp/irl_bench_nccl.{os.getpid()}.log")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    from paper_2601_17561_b200.ccmm import CcmmEngine, staging_tensors, synth_query
    from paper_2601_17561_b200.dist import PartRange, ShardedStep, deal_blocks, part_range
    from paper_2601_17561_b200.modmat import Context, build_paper_basis

    basis = build_paper_basis()
    nmod = len(basis.moduli)
    N = args.eyes * args.rot
    K = args.k
    # Dealing: whole parts (the paper's 8-slice layout), or balanced row blocks
    # when the b-parts are taller than the a-part (c5). Either way
    # the engine holds `local_parts.count` units of M rows; unit_map[j] is the
    # (global part, first row) of local unit j, a_units the owner's a-part units.
    use_blocks = args.deal == "blocks" or (args.deal == "auto" and args.b_rows != args.rows)
    if use_blocks:
        bd = deal_blocks(rank, world, args.rows, args.b_rows, args.parts)
        # every rank sizes its a-part buffer by the a-part's block count
        M, local_parts, unit_map, a_units = bd.block, PartRange(bd.first, bd.count), list(bd.blocks), args.rows // bd.block
    else:
        M = args.rows
        local_parts = part_range(rank, world, args.parts)
        unit_map, a_units = [(p, 0) for p in local_parts], 1
    ctx = Context(local)
    eng = CcmmEngine(parts=local_parts.count, m=M, k=K, max_n=N, basis=basis, ctx=ctx)
    if use_blocks:
        for j, (gp, r0) in enumerate(unit_map):
            eng.synth_part(j, args.seed, gp, r0)
    else:
        eng.synth_db(seed=args.seed, first_part=local_parts.first)
    moduli = eng.moduli
    q_host = synth_query(2, K, N, moduli)
    q_pinned = torch.from_numpy(q_host.view(np.int16)).pin_memory()
    q_dev, out_dev = staging_tensors(eng, N)
    q_dev.copy_(q_pinned)
    torch.cuda.synchronize()
    # ---- a-part exchange -------------------------------------
    # "mirror": receivers export an engine-owned receive buffer (CUDA IPC); the
    # owner's a-part PPMM epilogue stores every tile into all of them over
    # NVLink while it computes. Falls back to the NCCL broadcast when peer
    # mapping fails or the warm-up checksum disagrees.
    a_recv = None
    exchange, exch_note = "broadcast", None
    md_drop = max(0, min(args.moddown, nmod - 1))
    # --moddown: the step ends with the rescaled outputs [part][nmod - drop][N][M]
    # (f2), and the a-part exchange carries the rescaled copy
    out_md = (torch.empty((local_parts.count, nmod - md_drop, N, M), dtype=torch.int16, device="cuda")
              if md_drop else None)
    if world > 1:
        if args.exchange != "broadcast" and not md_drop:
            handle = None
            try:
                if rank != 0:
                    a_recv, handle = eng.alloc_recv(N, parts=a_units)
            except Exception as ex:  # noqa: BLE001
                exch_note = f"receive buffer: {ex}"
            handles = [None] * world
            dist.all_gather_object(handles, handle)
            ok = all(h is not None for r, h in enumerate(handles) if r != 0)
            if ok and rank == 0:
                try:
                    eng.set_mirrors(0, N, [h for r, h in enumerate(handles) if r != 0])
                    if a_units > 1:
                        eng.set_mirror_parts(a_units)
                except Exception as ex:  # noqa: BLE001
                    ok, exch_note = False, f"peer mapping: {ex}"
            flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 1:
                exchange = "mirror"
            elif rank == 0:
                eng.set_mirrors(0, N, [])
        if rank != 0 and a_recv is None:
            a_recv = torch.empty((2, a_units, nmod - md_drop, N, M), dtype=torch.int16, device="cuda")
    # The a-part receive buffers are double-buffered ([2] slots, alternating per
    # step): the owner's step s+1 stores into the other slot, so a consumer of
    # step s on a peer is never overwritten mid-read (irl_ccmm_set_mirror_slot).
    slot = [1]

    def next_slot():
        slot[0] ^= 1
        if world > 1 and rank == 0 and exchange == "mirror":
            eng.set_mirror_slot(slot[0])
    # a dedicated stream: the engine runs on the stream it is handed, and the
    # CUDA events below are recorded on that same stream
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    gemm_events = []

    def run_parts(first_local, count):
        # split the query into digit planes once per step (before the first
        # local PPMM), then time the PPMM launch itself for the roofline
        if first_local == 0:
            eng.run_device(None, N, None, part0=0, nparts=0, q_ready=False, stream=stream.cuda_stream)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.run_device(None, N, None, part0=first_local, nparts=count, q_ready=True, stream=stream.cuda_stream)
        e1.record(stream)
        gemm_events.append((e0, e1, count))
        if md_drop:
            eng.rescale(N, out_md[first_local:first_local + count], md_drop, True, part0=first_local,
                        nparts=count, stream=stream.cuda_stream)

    def a_out():
        if rank != 0:
            return a_recv[slot[0]]
        return out_md[:a_units] if md_drop else out_dev[:a_units]

    def make_step(kind):
        return ShardedStep(rank, world, run_parts, a_out, parts=args.parts, exchange=kind,
                           local=PartRange(0, local_parts.count) if use_blocks else None, a_parts=a_units)

    step = make_step(exchange)
    step_events = []

    def one_step():
        next_slot()
        w = step()
        if w is not None:
            w.wait()
        if world > 1:  # the exchange's completion on this rank's stream
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            step_events.append(ev)

    def a_checksum():
        # sum + exact head/tail samples of this rank's copy of the a-part result
        buf = a_out()
        flat = buf.view(-1)
        return torch.cat([torch.sum(buf.to(torch.int32), dtype=torch.int64).view(1),
                          flat[:512].to(torch.int64), flat[-512:].to(torch.int64)])

    if exchange == "mirror":
        # validate the fused exchange once before timing; fall back if any
        # receiver's copy differs from the owner's
        one_step()
        torch.cuda.synchronize()
        mine = a_checksum()
        src = mine.clone()
        dist.broadcast(src, src=0)
        flag = torch.tensor([1 if torch.equal(mine, src) else 0], dtype=torch.int32, device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) != 1:
            exchange, exch_note = "broadcast", "warm-up checksum mismatch on a receiver"
            if rank == 0:
                eng.set_mirrors(0, N, [])
            step = make_step(exchange)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    gemm_events.clear()
    step_events.clear()
    if world > 1:
        dist.barrier()
    launches0 = ctx.launches
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        t_start.record(stream)
        for _ in range(args.steps):
            one_step()
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = ctx.launches - launches0
    ms = t_start.elapsed_time(t_end) / args.steps
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_ops = 6.0 * nmod * total_rows(args) * N * K
    # per-rank breakdown of the timed steps: local GEMM launches, and the wait
    # from the last local GEMM to the exchange's completion on this rank
    per_rank = None
    if world > 1:
        runs = len(gemm_events) // max(1, args.steps)
        mine = {"rank": rank, "parts": [local_parts.first, local_parts.count], "step_ms": ms,
                "gemm_ms": sum(a.elapsed_time(b) for a, b, _ in gemm_events) / args.steps,
                "exchange_wait_ms": statistics.mean(
                    gemm_events[(i + 1) * runs - 1][1].elapsed_time(step_events[i]) for i in range(args.steps))
                if runs and len(step_events) == args.steps else None}
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    value = total_ops / (ms_max * 1e-3) / 1e12

    # dominant kernel: the PPMM launch (split is fused into the first launch's
    # stream slot but measured separately below)
    g_ms = [a.elapsed_time(b) for a, b, _ in gemm_events]
    g_parts = [c for _, _, c in gemm_events]
    ops_per_part = 6.0 * nmod * M * N * K
    launch_ops = statistics.mean(g_parts) * ops_per_part
    launch_ms = statistics.mean(g_ms)
    achieved = launch_ops / (launch_ms * 1e-3) / 1e12
    peaks = {}
    pk_path = ROOT / "MEASURED_PEAKS.json"
    if pk_path.exists():
        peaks = json.loads(pk_path.read_text())
    if "bf16_tflops_sustained" in peaks:
        peak = 2.0 * float(peaks["bf16_tflops_sustained"])
        peak_src = "2 x measured cuBLAS bf16 sustained (MEASURED_PEAKS.json); int8 dense = 2x bf16 dense on sm_100"
    else:
        peak = 2.0 * 1400.0
        peak_src = "2 x fallback bf16 sustained 1.4 PF/s (B200_PROFILING.md)"
    # roofline.traffic: ncu DRAM bytes of the PPMM (profiles/ppmm_traffic.json,
    # from the capture named there), scaled to this launch's parts; flagged
    # stale when the kernel source changed since that capture
    traffic, traffic_src = None, None
    tr_path = ROOT / "profiles" / "ppmm_traffic.json"
    if tr_path.exists():
        import hashlib
        tr = json.loads(tr_path.read_text())
        if (M, K, N) == (1 << 14, 24576, 992):  # the captured geometry (one c4 slice per part)
            traffic = tr.get("bytes_per_part", 0) * statistics.mean(g_parts) or None
        cur = hashlib.sha256((ROOT / "paper_2601_17561_b200" / "csrc" / "ppmm_gemm.cu").read_bytes()).hexdigest()
        traffic_src = {"capture": tr.get("source"), "per_part_bytes": tr.get("bytes_per_part"),
                       "algorithmic_per_part": tr.get("algorithmic_bytes_per_part"),
                       "kernel_source_matches_capture": tr.get("kernel_source_sha256") == cur}

    hbm_peak = float(peaks.get("hbm_gbs", 6457.4))
    R = SimpleNamespace(
        args=args, torch=torch, dist=dist, eng=eng, ctx=ctx, N=N, M=M, K=K, nmod=nmod, stream=stream,
        world=world, rank=rank, local_parts=local_parts, out_dev=out_dev, q_dev=q_dev, q_pinned=q_pinned,
        q_host=q_host, moduli=moduli, a_out=a_out, exchange=exchange, md_drop=md_drop, out_md=out_md,
        total_ops=total_ops, peaks=peaks, hbm_peak=hbm_peak, next_slot=next_slot, unit_map=unit_map,
        use_blocks=use_blocks)
    split_roof = measure_split(R)
    ingest = measure_ingest(R)
    moddown = measure_moddown(R)
    e2e = measure_e2e(R)
    dist_check = measure_dist_check(R)
    cpu = measure_cpu(R)
    fold = measure_fold(R)
    iris = measure_iris(R)
    int8_ref = measure_int8(R)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "int8 digits, int32 accumulate",
                "data": "synthetic residues (counter RNG, uniform mod p^2)",
                "config": config_dict(args, nmod),
                "ccmm_latency_ms": ms_max,
                "tensor_peak_frac": value / peak,
                "tensor_peak_frac_datasheet": value / DATASHEET_INT8_TOPS,
                "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS",
                             "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                             "kernel": "ppmm_i8_sm100_kernel", "launch_ms": launch_ms,
                             "ops_per_launch": launch_ops, "peak_source": peak_src,
                             "frac_of_datasheet_4500": achieved / DATASHEET_INT8_TOPS,
                             "frac_of_2x_bf16_burst": (achieved / (2.0 * float(peaks["bf16_tflops"]))
                                                       if "bf16_tflops" in peaks else None),
                             "frac_of_live_cublas_int8": (achieved / int8_ref["sustained_tops"]
                                                          if int8_ref else None)},
                "split_roofline": split_roof, "ingest": ingest, "moddown": moddown, "fold_stage": fold,
                "iris_stage": iris,
                "int8_library_ref": int8_ref,
                "dealing": ({"kind": "row blocks (dist.deal_blocks)", "block_rows": M,
                             "units_per_rank": [x["parts"][1] for x in per_rank] if per_rank else [local_parts.count]}
                            if use_blocks else {"kind": "whole parts (dist.part_range)"}),
                "exchange": None if world == 1 else {
                    "kind": "fused P2P stores in the a-part PPMM epilogue (CUDA IPC, NVLink)" if exchange == "mirror"
                    else "NCCL broadcast after the local GEMMs", "note": exch_note,
                    "bytes": int(a_out().numel() * 2)},
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "dist_check": dist_check,
                "per_rank": per_rank, "nccl": nccl_summary(nccl_log, world),
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""bench.py pieces that run on CPU: the reference arm (which must load only
oracle/ libraries, never the product package) and the NCCL log summary."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_loads_only_oracle_libraries():
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2", "--warmup", "1",
           "--cpu-rows", "2", "--k", "512", "--eyes", "2", "--rot", "4", "--rows", "64"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["product_package_imported"] is False
    assert d["loaded_repo_libs"] and all(p.startswith("oracle/") for p in d["loaded_repo_libs"])
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["host_cpu"]["threads_usable"] >= 1
    # the step is the bounded sample actually timed, not the extrapolation
    assert d["ms_per_step"] < 60_000 and d["ccmm_latency_ms_extrapolated"] > 0


def test_nccl_summary_parses_the_debug_log(tmp_path):
    sys.path.insert(0, str(ROOT))
    from bench import nccl_summary
    log = tmp_path / "nccl.log"
    log.write_text("host:1:1 [0] NCCL INFO NCCL version 2.28.9+cuda12.8\n"
                   "host:1:1 [0] NCCL INFO NVLS multicast support is available on dev 0\n"
                   "host:1:1 [0] NCCL INFO comm 0x5 rank 0 nranks 8 cudaDev 0 nvmlDev 0 busId 1000 commId 0x1 - "
                   "Init COMPLETE\n")
    s = nccl_summary(str(log), 8)
    assert s["nranks_seen"] == [8] and s["nvls"] is True and s["version"].startswith("2.28.9")
    assert nccl_summary(str(log), 1) is None
    assert nccl_summary(str(tmp_path / "missing.log"), 8)["read"] is False

"""The N>1 code paths of bench.py (part dealing, the fused a-part exchange over
CUDA IPC with its warm-up checksum validation, the completion signal, the e2e
loop, max-over-ranks timing) on a one-GPU box: torchrun with every rank on
GPU 0 and the gloo backend (IPC between processes of one device is legal).
The 8-GPU NCCL run is the driver's; this pins its logic."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("world,exchange", [(2, "auto"), (2, "broadcast"), (4, "auto"), (8, "auto")])
def test_bench_multirank_same_device(world, exchange):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", str(ROOT / "bench.py"), "--gpus", str(world),
           "--steps", "2", "--warmup", "3", "--backend", "gloo", "--same-device", "--parts", str(max(4, world)),
           "--rows", "2048",
           "--k", "4096", "--no-int8-ref", "--exchange", exchange]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 prints one JSON line
    d = json.loads(lines[0])
    assert d["n_gpus"] == world and d["steps"] == 2
    assert d["exchange"]["kind"].startswith("fused" if exchange == "auto" else "NCCL")
    assert d["exchange"]["note"] is None
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["e2e"]["outputs_equal_device_step"]
    assert d["dist_check"]["bit_exact_all_ranks"]  # sampled rows of every rank vs the CPU oracle
    # per-rank breakdown (diagnosable scaling runs): every rank's GEMM time and
    # its wait for the exchange after its last local GEMM
    pr = d["per_rank"]
    assert [x["rank"] for x in pr] == list(range(world))
    assert all(x["gemm_ms"] > 0 and x["exchange_wait_ms"] is not None for x in pr)
    assert sum(x["parts"][1] for x in pr) == max(4, world)
    # e2e per rank, with the sharded query distribution timed (H2D slice + all-gather)
    pe = d["e2e"]["per_rank"]
    assert [x["rank"] for x in pe] == list(range(world))
    assert all(x["e2e_ms"] > 0 and x["query_in_ms"] is not None and x["query_in_ms"] > 0 for x in pe)


@pytest.mark.gpu
def test_bench_multirank_moddown_exchange():
    """--moddown 3: every rank rescales its outputs to Q/Delta inside the step
    and the a-part broadcast carries the 21-modulus result (f2: "shrinks the
    broadcast"); all ranks end with the same a-part."""
    world = 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", str(ROOT / "bench.py"), "--gpus", str(world),
           "--steps", "2", "--warmup", "3", "--backend", "gloo", "--same-device", "--parts", "4",
           "--rows", "2048", "--k", "4096", "--no-int8-ref", "--moddown", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["config"]["moddown_drop"] == 3
    assert d["exchange"]["kind"].startswith("NCCL") and d["exchange"]["bytes"] == 21 * 31 * 32 * 2048 * 2
    assert d["dist_check"]["bit_exact_all_ranks"] and d["dist_check"]["a_part_identical_all_ranks"]
    assert d["e2e"]["outputs_equal_device_step"]


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", ["auto", "broadcast"])
def test_bench_multirank_row_blocks(exchange):
    """b-parts taller than the a-part (c5's shape, scaled down): balanced
    row-block dealing (dist.deal_blocks), the a-part spanning several blocks on
    rank 0 and mirrored / broadcast as a whole; every rank bit-exact."""
    world = 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", str(ROOT / "bench.py"), "--gpus", str(world),
           "--steps", "2", "--warmup", "3", "--backend", "gloo", "--same-device", "--parts", "4",
           "--rows", "2048", "--b-rows", "8192", "--k", "4096", "--no-int8-ref", "--exchange", exchange]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["dealing"]["kind"].startswith("row blocks") and d["dealing"]["block_rows"] == 512
    assert d["dealing"]["units_per_rank"] == [26, 26]   # (4 + 3 * 16) blocks of 512 rows
    assert d["exchange"]["note"] is None and d["exchange"]["bytes"] == 4 * 24 * 31 * 32 * 512 * 2
    assert d["dist_check"]["bit_exact_all_ranks"] and d["dist_check"]["a_part_identical_all_ranks"]
    assert d["e2e"]["outputs_equal_device_step"]
    assert d["config"]["templates_per_b_part"] == 8192

"""Multi-rank layout of the CCMM (paper's 8-slice DB, a-part broadcast) on CPU
with the gloo backend. The per-part PPMM is stood in by the CPU oracle (test
infrastructure) so the orchestration (part dealing, broadcast ordering, result
placement) is exercised exactly as bench.py drives it on NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as ol
from paper_2601_17561_b200.dist import PAPER_PARTS, ShardedStep, a_part_owner, part_range

M, K, N = 40, 96, 12
MODS = [127 * 127, 251 * 251]
SEED = 3


def test_part_ranges_cover_db_once():
    for world in (1, 2, 4, 8, 3, 5):
        seen = []
        for r in range(world):
            seen += list(part_range(r, world))
        assert sorted(seen) == list(range(PAPER_PARTS))
        assert a_part_owner(world) == 0
    assert [part_range(r, 8).count for r in range(8)] == [1] * 8
    assert [part_range(r, 2).first for r in range(2)] == [0, 4]
    with pytest.raises(ValueError):
        part_range(0, 9)


def oracle_part(part, q):
    out = np.zeros((len(MODS), N, M), np.uint16)
    for i, m in enumerate(MODS):
        a = ol.synth_block(SEED, part, i, 0, M, 0, K, m)
        out[i] = ol.ppmm_rows_direct(a, np.ascontiguousarray(q[i].T), np.arange(M, dtype=np.uint32), m).T
    return out


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q = np.stack([ol.synth_block(9, 0xFF, i, 0, K, 0, N, m) for i, m in enumerate(MODS)])
    local = part_range(rank, world)
    out = torch.zeros((local.count, len(MODS), N, M), dtype=torch.int16)
    a_recv = torch.zeros((len(MODS), N, M), dtype=torch.int16)
    calls = []

    def run_parts(first_local, count):
        calls.append((first_local, count))
        for g in range(first_local, first_local + count):
            out[g] = torch.from_numpy(oracle_part(local.first + g, q).view(np.int16))

    def a_out():
        return out[0] if rank == a_part_owner(world) else a_recv

    step = ShardedStep(rank, world, run_parts, a_out)
    w = step()
    if w is not None:
        w.wait()
    ok_local = all((out[g].numpy().view(np.uint16) == oracle_part(local.first + g, q)).all()
                   for g in range(local.count))
    ok_a = bool((a_out().numpy().view(np.uint16) == oracle_part(0, q)).all())
    results[rank] = (ok_local, ok_a, calls)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_step_gloo(world):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert sorted(results.keys()) == list(range(world))
    for r in range(world):
        ok_local, ok_a, calls = results[r]
        assert ok_local and ok_a, r
        if r == 0:
            # the a-part GEMM is issued first, then the b-parts; the broadcast
            # is posted once every local GEMM is queued
            assert calls[0] == (0, 1)


def _worker_mirror(rank, world, port, results):
    # exchange="mirror": no broadcast; the step posts a 4-byte all-reduce as the
    # completion signal (the data itself moves inside the owner's GEMM epilogue,
    # stood in here by the owner copying into a shared-memory "peer" buffer)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []
    buf = torch.zeros(4, dtype=torch.int16)

    def run_parts(first_local, count):
        calls.append((first_local, count))

    step = ShardedStep(rank, world, run_parts, lambda: buf, exchange="mirror")
    w = step()
    w.wait()
    results[rank] = (calls, int(step._flag.item()))
    dist.destroy_process_group()


def test_sharded_step_mirror_signal_gloo():
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker_mirror, args=(2, _free_port(), results), nprocs=2, join=True)
    assert results[0][0] == [(0, 1), (1, 3)] and results[1][0] == [(0, 4)]
    assert results[0][1] == 0 and results[1][1] == 0
    with pytest.raises(ValueError):
        ShardedStep(0, 1, lambda a, b: None, lambda: None, exchange="nccl")


# ---------------------------------------------- row-block dealing (c5) -------

def test_deal_blocks_balanced_and_complete():
    from paper_2601_17561_b200.dist import deal_blocks
    for a_rows, b_rows in [(1 << 14, 1 << 17), (1 << 14, 1 << 15), (2048, 8192), (1 << 14, 1 << 14)]:
        for world in (1, 2, 3, 4, 8):
            deals = [deal_blocks(r, world, a_rows, b_rows) for r in range(world)]
            block = deals[0].block
            assert block % 256 == 0 and a_rows % block == 0 and b_rows % block == 0
            got = [b for d in deals for b in d.blocks]
            want = [(0, r) for r in range(0, a_rows, block)] + \
                   [(p, r) for p in range(1, PAPER_PARTS) for r in range(0, b_rows, block)]
            assert got == want                                   # every row once, in order
            counts = [d.count for d in deals]
            assert max(counts) - min(counts) <= 1                # balanced to one block
            assert deals[0].a_blocks == a_rows // block          # the a-part stays on rank 0
            assert all(d.a_blocks == 0 for d in deals[1:])
            assert deals[0].locate(0, a_rows - 1) == (a_rows // block - 1, block - 1)
    # c5 on 8 GPUs: the largest share falls from a whole 2^17-row b-part to
    # 29 blocks of 4096 rows (the even split is 116736 rows)
    c5 = [deal_blocks(r, 8, 1 << 14, 1 << 17) for r in range(8)]
    assert max(d.count * d.block for d in c5) == 118784 < (1 << 17)


def _worker_blocks(rank, world, port, results):
    # ShardedStep over row blocks: the owner runs its a-part blocks first, and
    # the broadcast carries all of them
    from paper_2601_17561_b200.dist import PartRange, deal_blocks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bd = deal_blocks(rank, world, 512, 1024, parts=4, block=256)
    calls = []
    out = torch.zeros((bd.count, 4), dtype=torch.int32)
    a_units = max(1, bd.a_blocks)
    recv = torch.zeros((a_units if rank == 0 else 2, 4), dtype=torch.int32)

    def run_parts(first_local, count):
        calls.append((first_local, count))
        for j in range(first_local, first_local + count):
            gp, r0 = bd.blocks[j]
            out[j] = torch.tensor([gp, r0, rank, 7], dtype=torch.int32)

    def a_out():
        return out[:a_units] if rank == 0 else recv

    step = ShardedStep(rank, world, run_parts, a_out, local=PartRange(0, bd.count), a_parts=a_units)
    step().wait()
    results[rank] = (calls, bd.count, recv.tolist() if rank else out[:a_units].tolist())
    dist.destroy_process_group()


def test_sharded_step_row_blocks_gloo():
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker_blocks, args=(2, _free_port(), results), nprocs=2, join=True)
    # 2 + 3 * 4 = 14 blocks of 256 rows: 7 per rank; rank 0 runs its 2 a-part blocks first
    assert results[0][0] == [(0, 2), (2, 5)] and results[1][0] == [(0, 7)]
    assert results[0][1] == results[1][1] == 7
    assert results[1][2] == results[0][2] == [[0, 0, 0, 7], [0, 256, 0, 7]]

"""Multi-GPU layout of the RGSW CCMM (reference cost model
proj/src/costmodel.cpp:59-73).

The database is the paper's 8 slices: part 0 is the shared a-part, parts
1..7 are b-part slices of 2^14 templates. Parts are independent PPMMs against
the same query, so they are dealt to ranks with no data-path collective; the
one real exchange is the broadcast of the a-part result from its
owner (rank 0) to every rank, so each rank can assemble (out_A, out_B,i) score
ciphertexts. One process per GPU; NCCL via torch.distributed is the plumbing.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

PAPER_PARTS = 8
A_PART = 0


@dataclass(frozen=True)
class PartRange:
    first: int
    count: int

    def __iter__(self):
        return iter(range(self.first, self.first + self.count))


def part_range(rank: int, world: int, parts: int = PAPER_PARTS) -> PartRange:
    """Contiguous block of parts for `rank` (1/2/4/8 GPUs: 8/4/2/1 parts each).
    Uneven worlds get ceil/floor blocks; the a-part always lands on rank 0."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if world > parts:
        raise ValueError(f"at most {parts} ranks for {parts} parts")
    base, extra = divmod(parts, world)
    first = rank * base + min(rank, extra)
    return PartRange(first, base + (1 if rank < extra else 0))


@dataclass(frozen=True)
class BlockDeal:
    """Row-block dealing (SURVEY 8(e) imbalance note): the global database is
    the a-part (a_rows rows) followed by parts-1 b-parts of b_rows rows, cut
    into blocks of `block` rows; rank r holds the contiguous global blocks
    [first, first + count). blocks[j] = (global part, first row) of local block
    j. The a-part's blocks are the first a_blocks blocks, always on rank 0."""
    block: int
    first: int
    count: int
    blocks: tuple
    a_blocks: int      # leading local blocks that belong to the a-part (rank 0 only)

    def locate(self, part: int, row: int):
        """(local block, row within it) of global (part, row), or None."""
        for j, (p, r0) in enumerate(self.blocks):
            if p == part and r0 <= row < r0 + self.block:
                return j, row - r0
        return None


def block_rows(a_rows: int, b_rows: int, world: int) -> int:
    """Block size for deal_blocks: a multiple of 256 rows (the PPMM's row
    block) dividing both part heights, small enough that the blocks spread
    evenly (a quarter of the shorter part, or 256)."""
    from math import gcd
    g = gcd(a_rows, b_rows)
    b = max(256, min(a_rows, b_rows) // 4)
    while b > 256 and g % b:
        b //= 2
    if g % b or b % 256:
        raise ValueError(f"part heights {a_rows}, {b_rows} need a common multiple-of-256 block")
    return b


def deal_blocks(rank: int, world: int, a_rows: int, b_rows: int, parts: int = PAPER_PARTS,
                block: int = 0) -> BlockDeal:
    """Balanced contiguous dealing of row blocks: rank r gets floor or ceil of
    T / world of the T blocks (b-parts taller than the a-part no longer leave
    rank 0 idle: at c5, 2^14 + 7 * 2^17 rows over 8 GPUs, the largest share is
    29 blocks of 4096 rows = 1.02x the even split, against 2^17 rows = 1.12x
    when whole parts are dealt)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    block = block or block_rows(a_rows, b_rows, world)
    if a_rows % block or b_rows % block:
        raise ValueError("block must divide both part heights")
    glob = [(0, r) for r in range(0, a_rows, block)]
    for p in range(1, parts):
        glob += [(p, r) for r in range(0, b_rows, block)]
    total = len(glob)
    if world > total:
        raise ValueError(f"at most {total} ranks for {total} blocks")
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    a_total = a_rows // block
    if rank == 0 and count < a_total:
        raise ValueError("rank 0 must hold the whole a-part (fewer ranks or smaller blocks)")
    mine = tuple(glob[first:first + count])
    return BlockDeal(block, first, count, mine, a_total if rank == 0 else 0)


def a_part_owner(world: int, parts: int = PAPER_PARTS) -> int:
    for r in range(world):
        if A_PART in part_range(r, world, parts):
            return r
    raise AssertionError


class ShardedStep:
    """One CCMM step on this rank.

    run_parts(first_local, count) launches the local PPMMs for local parts
    [first_local, first_local + count) (stream-ordered, non-blocking);
    a_out() returns this rank's buffer for the a-part result: on the owner it
    is the local output of part 0, elsewhere a receive buffer.

    Every rank posts the broadcast after its local GEMMs are queued. The
    PPMM is persistent and holds every SM (1 CTA per SM, 8-CTA clusters), and
    NCCL's broadcast kernels need SMs: a receive posted before the GEMM would
    park its CTAs on SMs for the whole step and knock whole clusters out of the
    GEMM, and an owner's send posted between its a-part and b-part GEMMs would
    wait on receivers in the same way. Posted last, the NCCL stream waits for
    the GEMMs and then runs the 744 MiB exchange with the whole GPU (~1 ms
    over NVLink, <= 5% of an 8-GPU step).

    exchange: "broadcast" (NCCL broadcast of the a-part result) or "mirror"
    (the owner's a-part PPMM epilogue already stored it into every peer's
    receive buffer over NVLink, irl_ccmm_set_mirrors; the step then only posts
    a 4-byte all-reduce so peers' later reads are ordered after the owner's
    GEMM).
    """

    def __init__(self, rank: int, world: int, run_parts: Callable[[int, int], None],
                 a_out: Callable[[], object], parts: int = PAPER_PARTS, group=None,
                 exchange: str = "broadcast", local: Optional[PartRange] = None, a_parts: int = 1):
        """local / a_parts: the rank's local units and how many leading ones
        hold the a-part on the owner (row-block dealing: deal_blocks)."""
        if exchange not in ("broadcast", "mirror"):
            raise ValueError(exchange)
        self.exchange = exchange
        self._flag = None
        self.rank, self.world = rank, world
        self.local = local if local is not None else part_range(rank, world, parts)
        self.a_parts = a_parts
        self.owner = 0 if local is not None else a_part_owner(world, parts)
        self.run_parts = run_parts
        self.a_out = a_out
        self.group = group

    def _bcast(self):
        import torch
        import torch.distributed as dist
        buf = self.a_out()
        # residues are uint16 bit patterns; exchange them as bytes (gloo and
        # NCCL both carry uint8)
        return dist.broadcast(buf.view(torch.uint8), src=self.owner, group=self.group, async_op=True)

    def _signal(self):
        import torch
        import torch.distributed as dist
        if self._flag is None:
            buf = self.a_out()
            self._flag = torch.zeros(1, dtype=torch.int32, device=buf.device)
        return dist.all_reduce(self._flag, group=self.group, async_op=True)

    def __call__(self):
        work = None
        if self.world > 1:
            if self.rank == self.owner:
                self.run_parts(0, self.a_parts)  # a-part first
                if self.local.count > self.a_parts:
                    self.run_parts(self.a_parts, self.local.count - self.a_parts)
            else:
                self.run_parts(0, self.local.count)
            work = self._bcast() if self.exchange == "broadcast" else self._signal()
        else:
            self.run_parts(0, self.local.count)
        return work

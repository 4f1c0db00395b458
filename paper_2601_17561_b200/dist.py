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
                 exchange: str = "broadcast"):
        if exchange not in ("broadcast", "mirror"):
            raise ValueError(exchange)
        self.exchange = exchange
        self._flag = None
        self.rank, self.world = rank, world
        self.local = part_range(rank, world, parts)
        self.owner = a_part_owner(world, parts)
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
                self.run_parts(0, 1)  # a-part first
                if self.local.count > 1:
                    self.run_parts(1, self.local.count - 1)
            else:
                self.run_parts(0, self.local.count)
            work = self._bcast() if self.exchange == "broadcast" else self._signal()
        else:
            self.run_parts(0, self.local.count)
        return work

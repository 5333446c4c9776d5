"""Multi-GPU PaLD: one process per GPU, torch.distributed (NCCL) plumbing.

Work decomposition:
  * D is replicated (every rank lays out the same fp32 matrix).
  * Pass 1 (focus): the work units (upper-triangular 128x128 pair tile x
    64-point chunk of third points) are split into equal contiguous shares,
    one per rank (exact balance; the reference's analogue is the z-split of
    parallel.hpp:185-204 with private partial counts summed). Each rank
    accumulates integer focus counts; one SUM all-reduce of the count
    buffer (exact: integers < 2^24 in fp32) and a local finish give every
    rank the full U and W = 1/U.
  * Pass 2 (cohesion): the engine's cohesion_share(rank, world) computes an
    equal share of the pass-2 work into a zeroed C -- contiguous ranges of
    the tile-pair list on the pair kernel (each pair writes C[P][Q] and
    C[Q][P]), tile-row bands on the one-sided kernel. Every C entry is one
    complete in-order sum on exactly one rank (bit-identical to 1 GPU) and
    0 on the others, so one SUM all-reduce of C assembles it exactly.
The exchange steps are real data dependencies (W between the passes, C at
the end); nothing else crosses ranks. ``cohesion_row_split`` / the row-band
all-gather remain for engines without cohesion_share.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def cohesion_row_split(n: int, tile: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, tile-aligned row bands [r0, r1) of ~equal pass-2 work."""
    nb = (n + tile - 1) // tile
    per = -(-nb // world)  # ceil
    out = []
    for k in range(world):
        t0, t1 = min(nb, k * per), min(nb, (k + 1) * per)
        out.append((min(n, t0 * tile), min(n, t1 * tile)))
    return out


@dataclass
class ShardPlan:
    rank: int
    world: int
    focus_share: tuple[int, int]      # (part, parts) of the pass-1 work units
    cohesion_rows: tuple[int, int]
    band_rows: int  # padded rows per rank for the C all-gather


def make_shard_plan(n: int, tile: int, rank: int, world: int) -> ShardPlan:
    c = cohesion_row_split(n, tile, world)
    band = max(r1 - r0 for r0, r1 in c)
    return ShardPlan(rank, world, (rank, world), c[rank], band)


class ShardedRunner:
    """Runs one full PaLD step across the ranks of ``group``.

    ``engine`` is a paper_2307_16652_b200.engine.Engine (or any object with
    the same load / focus / cohesion / full_U / full_W / row_block_C / C
    interface -- the CPU tests use a gloo-backed stand-in).
    """

    def __init__(self, engine, group=None):
        self.engine = engine
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.plan = make_shard_plan(engine.n, engine.tile, self.rank, self.world)
        ld = engine.ld
        self._even = all(r1 - r0 == self.plan.band_rows
                         for r0, r1 in cohesion_row_split(engine.n, engine.tile, self.world))
        self._even = self._even and self.plan.band_rows * self.world == engine.n
        if not self._even:
            dev = engine.C.device
            self._send = torch.zeros(self.plan.band_rows * ld, dtype=torch.float32, device=dev)
            self._recv = torch.empty(self.world * self.plan.band_rows * ld, dtype=torch.float32, device=dev)

    def exchange_focus(self) -> None:
        """SUM the integer focus counts over ranks, then finish locally."""
        if self.world > 1:
            dist.all_reduce(self.engine.full_W(), op=dist.ReduceOp.SUM, group=self.group)
        self.engine.focus_finish()

    def reduce_cohesion(self) -> None:
        """SUM of the per-rank C shares (disjoint supports: exact)."""
        if self.world > 1:
            e = self.engine
            dist.all_reduce(e.row_block_C(0, e.n), op=dist.ReduceOp.SUM, group=self.group)

    def gather_cohesion(self) -> None:
        if self.world == 1:
            return
        e, p = self.engine, self.plan
        r0, r1 = p.cohesion_rows
        if self._even:
            full = e.row_block_C(0, e.n)
            dist.all_gather_into_tensor(full, e.row_block_C(r0, r1), group=self.group)
            return
        ld = e.ld
        self._send.zero_()
        if r1 > r0:
            self._send[: (r1 - r0) * ld].copy_(e.row_block_C(r0, r1))
        dist.all_gather_into_tensor(self._recv, self._send, group=self.group)
        for k, (a, b) in enumerate(cohesion_row_split(e.n, e.tile, self.world)):
            if b > a:
                src = self._recv[k * p.band_rows * ld: k * p.band_rows * ld + (b - a) * ld]
                e.row_block_C(a, b).copy_(src)

    def cohesion(self, stream=None) -> None:
        """This rank's share of pass 2."""
        e = self.engine
        if getattr(e, "cohesion_share", None) is not None:
            e.cohesion_share(self.rank, self.world, stream=stream)
        else:
            e.cohesion(*self.plan.cohesion_rows, stream=stream)

    def assemble_cohesion(self) -> None:
        """Full C on every rank: SUM all-reduce of the shares (or the
        row-band all-gather for engines without cohesion_share)."""
        if getattr(self.engine, "cohesion_share", None) is not None:
            self.reduce_cohesion()
        else:
            self.gather_cohesion()

    def step(self, D, stream=None) -> None:
        e, p = self.engine, self.plan
        e.load(D, stream)
        e.focus_counts(*p.focus_share, stream=stream)
        self.exchange_focus()
        self.cohesion(stream=stream)
        self.assemble_cohesion()

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
the end); nothing else crosses ranks.

Fused mode (``fused=True``, the default for N > 1 when the engine supports
it): the two all-reduces are replaced by the kernels themselves writing over
NVLink into every rank's buffers (CUDA IPC mappings, include/pald_gpu.h):
pass-1 partial counts are added into every rank's W and the pair kernel
stores each C entry into every rank's C. The host orders the ranks with a
barrier after load (all W zeroed), after pass 1 (all counts in) and after
pass 2 (all of C written). If a rank cannot map its peers, every rank
falls back to the collectives; if the pair kernel does not run for the
loaded D (tie-heavy input, InclusiveSplit, exact path), pass 2 of that step
uses cohesion_share + the all-reduce. ``cohesion_row_split`` / the row-band
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

    def __init__(self, engine, group=None, fused: bool | None = None, focus_exchange: str | None = None,
                 cohesion_exchange: str | None = None):
        """``focus_exchange`` (pass 1): "peer" (peer-pull finish over the
        mapped buffers, the default when mapping works), "red" (partial
        counts added into every rank's W by the focus kernel) or "nccl" (SUM
        all-reduce of the counts). ``cohesion_exchange`` (pass 2): "peer"
        (the pair kernel stores into every rank's C, default when mapping
        works) or "nccl" (SUM all-reduce of the C shares). ``fused=False``
        forces "nccl" for both."""
        self.engine = engine
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.plan = make_shard_plan(engine.n, engine.tile, self.rank, self.world)
        self.fused = False
        self._fused_c = False  # this step's pass 2 ran fused
        for x, ok in ((focus_exchange, ("peer", "red", "nccl", None)), (cohesion_exchange, ("peer", "nccl", None))):
            if x not in ok:
                raise ValueError(f"unknown exchange {x!r}")
        if fused is None:
            fused = self.world > 1 and hasattr(engine, "attach_peers")
        if fused and self.world > 1:
            self.fused = self._attach_peers(need_u=(focus_exchange or "peer") == "peer")
        self.focus_exchange = (focus_exchange or "peer") if self.fused else "nccl"
        self.cohesion_exchange = (cohesion_exchange or "peer") if self.fused else "nccl"
        ld = engine.ld
        self._even = all(r1 - r0 == self.plan.band_rows
                         for r0, r1 in cohesion_row_split(engine.n, engine.tile, self.world))
        self._even = self._even and self.plan.band_rows * self.world == engine.n
        if not self._even:
            dev = engine.C.device
            self._send = torch.zeros(self.plan.band_rows * ld, dtype=torch.float32, device=dev)
            self._recv = torch.empty(self.world * self.plan.band_rows * ld, dtype=torch.float32, device=dev)

    def _attach_peers(self, need_u: bool = True) -> bool:
        """Map every rank's W and C (and U for the peer-pull finish) into this
        process; all ranks agree on the outcome (any failure -> collectives
        everywhere)."""
        ok = 1
        try:
            mine = self.engine.export_buffers() + ((self.engine.export_u(),) if need_u else (b"",))
        except Exception:
            mine, ok = (b"", b"", b""), 0
        handles = [None] * self.world
        dist.all_gather_object(handles, mine, group=self.group)
        if ok and all(h[0] for h in handles):
            try:
                self.engine.attach_peers(self.rank, [h[0] for h in handles], [h[1] for h in handles])
                if need_u:
                    self.engine.attach_peers_u([h[2] for h in handles])
            except Exception:
                ok = 0
        else:
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=self._flag_device())
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        if int(flag.item()) == 0:
            if ok:
                self.engine.detach_peers()
            return False
        return True

    def _flag_device(self):
        backend = dist.get_backend(self.group)
        return self.engine.C.device if backend == "nccl" else "cpu"

    def _sync_barrier(self, stream=None) -> None:
        """Host barrier after this rank's work on `stream` (the stream the
        engine calls were issued on, default the current one) has finished."""
        (stream if stream is not None else torch.cuda.current_stream()).synchronize()
        dist.barrier(group=self.group)

    @staticmethod
    def _before_collective(stream) -> None:
        """Collectives run on the current stream: order them after the work
        issued on `stream`."""
        if stream is not None and torch.cuda.is_available():
            torch.cuda.current_stream().wait_stream(stream)

    @staticmethod
    def _after_collective(stream) -> None:
        """Order later work on `stream` after the collective."""
        if stream is not None and torch.cuda.is_available():
            stream.wait_stream(torch.cuda.current_stream())

    def _agree(self, flag: bool) -> bool:
        """True iff `flag` holds on every rank (MIN all-reduce)."""
        t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=self._flag_device())
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return bool(int(t.item()))

    def load(self, D, stream=None) -> None:
        self.engine.load(D, stream)
        if self.world > 1 and self.focus_exchange == "red":
            self._sync_barrier(stream)  # every rank's W zeroed before any rank adds into it

    def focus(self, stream=None) -> None:
        """This rank's share of pass 1 (counts into its W, or into every W)."""
        if self.world > 1 and self.focus_exchange == "red":
            self.engine.focus_counts_peers(*self.plan.focus_share, stream=stream)
        else:
            self.engine.focus_counts(*self.plan.focus_share, stream=stream)

    def exchange_focus(self, stream=None) -> None:
        """Combine the integer focus counts of the ranks and finish U / W."""
        if self.world == 1:
            self.engine.focus_finish(stream=stream)
        elif self.focus_exchange == "peer":
            self._sync_barrier(stream)  # every rank's counts are in its W
            self.engine.focus_finish_peers(self.rank, self.world, u_mode=1, stream=stream)
            self._sync_barrier(stream)  # every W (and U) finished everywhere
        elif self.focus_exchange == "red":
            self._sync_barrier(stream)  # all ranks' counts are in every W
            self.engine.focus_finish(stream=stream)
        else:
            self._before_collective(stream)
            dist.all_reduce(self.engine.full_W(), op=dist.ReduceOp.SUM, group=self.group)
            self._after_collective(stream)
            self.engine.focus_finish(stream=stream)

    def reduce_cohesion(self, stream=None) -> None:
        """SUM of the per-rank C shares (disjoint supports: exact)."""
        if self.world > 1:
            e = self.engine
            self._before_collective(stream)
            dist.all_reduce(e.row_block_C(0, e.n), op=dist.ReduceOp.SUM, group=self.group)
            self._after_collective(stream)

    def gather_cohesion(self, stream=None) -> None:
        if self.world == 1:
            return
        self._before_collective(stream)
        self._gather_cohesion()
        self._after_collective(stream)

    def _gather_cohesion(self) -> None:
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
        self._fused_c = False
        if self.world > 1 and self.cohesion_exchange == "peer":
            # The pair-kernel choice is made per rank (it depends on D and on
            # the device's SM count / env knobs): run fused only if every rank
            # can, decided BEFORE any rank stores into its peers' C.
            if self._agree(e.pair_kernel_preferred()):
                self._fused_c = e.cohesion_share_peers(self.rank, self.world, stream=stream)
                if not self._fused_c:
                    raise RuntimeError("fused pass 2 refused after all ranks agreed on the pair kernel")
                return
        if getattr(e, "cohesion_share", None) is not None:
            e.cohesion_share(self.rank, self.world, stream=stream)
        else:
            e.cohesion(*self.plan.cohesion_rows, stream=stream)

    def assemble_cohesion(self, stream=None) -> None:
        """Full C on every rank: a barrier after the fused pass 2, else the
        SUM all-reduce of the shares (or the row-band all-gather for engines
        without cohesion_share)."""
        if self.world == 1:
            return
        # every rank took the same branch (agreed in cohesion())
        if self._fused_c:
            self._sync_barrier(stream)
        elif getattr(self.engine, "cohesion_share", None) is not None:
            self.reduce_cohesion(stream)
        else:
            self.gather_cohesion(stream)

    def step(self, D, stream=None) -> None:
        self.load(D, stream)
        self.focus(stream=stream)
        self.exchange_focus(stream)
        self.cohesion(stream=stream)
        self.assemble_cohesion(stream)

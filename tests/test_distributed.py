"""Multi-rank path on CPU: world_size 2 (and 3) over gloo.

The sharded driver (paper_2307_16652_b200.distributed) runs unchanged; the
GPU engine is replaced by a CPU stand-in with the same staged interface
(load / focus / cohesion / cohesion_share / buffer views) whose arithmetic
is the oracle's restatement, so what is tested here is exactly the
decomposition and the exchange: unit shares of pass 1, SUM all-reduce of
the counts, tile-pair shares of pass 2 computed from the *exchanged* W and
the SUM all-reduce of C (or, for engines without cohesion_share, row bands
and the C all-gather).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import int_upper, random_upper


class CpuEngine:
    """CPU stand-in for paper_2307_16652_b200.engine.Engine."""

    def __init__(self, n: int, tile: int):
        self.n, self.tile = n, tile
        self.ld = n + 3  # exercise the leading dimension
        self.tiles_per_dim = (n + tile - 1) // tile
        self._u = torch.zeros(n * self.ld, dtype=torch.int32)
        self._w = torch.zeros(n * self.ld, dtype=torch.float32)
        self._c = torch.zeros(n * self.ld, dtype=torch.float32)
        self.d = None

    @property
    def U(self):
        return self._u.view(self.n, self.ld)[:, : self.n]

    @property
    def W(self):
        return self._w.view(self.n, self.ld)[:, : self.n]

    @property
    def C(self):
        return self._c.view(self.n, self.ld)[:, : self.n]

    def full_U(self):
        return self._u

    def full_W(self):
        return self._w

    def row_block_C(self, r0, r1):
        return self._c[r0 * self.ld: r1 * self.ld]

    def load(self, D, stream=None):
        self.d = D.numpy().astype(np.float32)
        self._u.zero_()
        self._w.zero_()

    BK = 4  # stand-in chunk of third points (the GPU uses 32)

    def focus_counts(self, part, parts, stream=None):
        """Integer focus counts of share `part` of `parts` of the units
        u = tile * nchunks + chunk over the upper-triangular tiles (the GPU
        engine's decomposition), accumulated into W."""
        d, n, T, nb = self.d, self.n, self.tile, self.tiles_per_dim
        tiles = [(tr, tc) for tr in range(nb) for tc in range(tr, nb)]
        nch = (n + self.BK - 1) // self.BK
        units = len(tiles) * nch
        W = self.W
        for u in range(units * part // parts, units * (part + 1) // parts):
            tr, tc = tiles[u // nch]
            k0, k1 = (u % nch) * self.BK, min(n, (u % nch + 1) * self.BK)
            for r in range(tr * T, min(n, tr * T + T)):
                for c in range(tc * T, min(n, tc * T + T)):
                    W[r, c] += float((np.minimum(d[r, k0:k1], d[c, k0:k1]) < d[r, c]).sum())

    def focus_finish(self, stream=None):
        n = self.n
        U, W = self.U, self.W
        cnt = W.numpy().copy()
        for r in range(n):
            U[r, r] = 0
            W[r, r] = 0.0
            for c in range(r + 1, n):
                u = int(cnt[r, c])
                U[r, c] = U[c, r] = u
                W[r, c] = W[c, r] = float(np.float32(1) / np.float32(u))

    def _cohesion_row(self, r):
        d, n = self.d, self.n
        w = self.W.numpy()
        dn = np.nextafter(d, np.float32(np.inf))
        acc = np.zeros(n, np.float32)
        for k in range(n):
            b = dn[k] if k < r else d[k]
            m = np.minimum(d[r, k], b)
            acc = np.where(d[r] < m, (acc + w[r, k]).astype(np.float32), acc)
        return acc

    def cohesion(self, r0, r1, stream=None):
        for r in range(r0, r1):
            self.C[r] = torch.from_numpy(self._cohesion_row(r))

    def cohesion_share(self, part, parts, stream=None):
        """The GPU engine's pair-kernel decomposition: zero C, then compute
        both C[P][Q] and C[Q][P] for the tile pairs (P <= Q) of share
        `part` of the upper-triangular pair list."""
        n, T, nb = self.n, self.tile, self.tiles_per_dim
        self._c.zero_()
        pairs = [(P, Q) for P in range(nb) for Q in range(P, nb)]
        full = np.stack([self._cohesion_row(r) for r in range(n)])
        C = self.C
        for P, Q in pairs[len(pairs) * part // parts: len(pairs) * (part + 1) // parts]:
            rp, rq = slice(P * T, min(n, P * T + T)), slice(Q * T, min(n, Q * T + T))
            C[rp, rq] = torch.from_numpy(full[rp, rq])
            C[rq, rp] = torch.from_numpy(full[rq, rp])


class CpuEngineRows(CpuEngine):
    """Stand-in without cohesion_share: the row-band all-gather path."""
    cohesion_share = None


def _worker(rank, world, port, n, tile, d, out, rows=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2307_16652_b200.distributed import ShardedRunner

    eng = CpuEngineRows(n, tile) if rows else CpuEngine(n, tile)
    runner = ShardedRunner(eng)
    runner.step(torch.from_numpy(d))
    out[rank] = (eng.U.numpy().copy(), eng.C.numpy().copy(), runner.plan)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,n,tile,kind,rows", [
    (2, 21, 4, "ties", False), (2, 16, 4, "rand", False), (3, 23, 4, "ties", False),
    (2, 21, 4, "ties", True), (3, 23, 4, "rand", True),
])
def test_sharded_equals_single(oracle, world, n, tile, kind, rows):
    d = int_upper(n, n) if kind == "ties" else random_upper(n, n)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, tile, d, out, rows), nprocs=world, join=True)
    u_ref, c_ref = oracle.pairwise_f32(d)
    covered = []
    for r in range(world):
        u, c, plan = out[r]
        assert np.array_equal(u, u_ref)
        assert np.array_equal(c.view(np.uint32), c_ref.view(np.uint32))
        covered.append(plan.cohesion_rows)
    assert covered[0][0] == 0 and covered[-1][1] == n


def test_row_split():
    from paper_2307_16652_b200.distributed import cohesion_row_split, make_shard_plan

    for n in (2, 100, 1000, 32768):
        for world in (1, 2, 4, 8):
            rows = cohesion_row_split(n, 128, world)
            assert rows[0][0] == 0 and rows[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            assert all(r0 % 128 == 0 for r0, r1 in rows if r1 > r0)
            plan = make_shard_plan(n, 128, world - 1, world)
            assert plan.focus_share == (world - 1, world)

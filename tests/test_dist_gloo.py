"""Multi-process (world_size 2, gloo, CPU) tests of the partitioner's host logic
(DESIGN.md §7): shard ranges, halo assembly from the orbit, all-gather order and the
orbit→g permutation.  The per-rank compute is a test double built from oracle primitives
that uses only the rank's stacked input blocks, so wrong halo/placement fails the test."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import blockperm as bp
from paper_2602_06071_b200 import dist as D


def test_column_shard_partition():
    for n in [1, 127, 128, 512, 1000, 4096]:
        for world in [1, 2, 3, 8]:
            rs = [D.column_shard(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            for (a, b), (c, _) in zip(rs, rs[1:]):
                assert b == c and a <= b and a % 128 == 0


def test_orbit_shard_and_halo():
    osk = oracle.make_sketch(1024, 16, 64, 8, 4, 1234)
    orbit = bp.orbit(osk.a, osk.b, osk.M)
    covered = []
    for r in range(8):
        p0, p1 = D.orbit_shard(1024, 8, r)
        covered += list(range(p0, p1))
        blocks = D.input_blocks(orbit, p0, p1, 8)
        assert len(blocks) == (p1 - p0) + 7
        # every output block's neighbourhood lies inside the rank's input blocks
        for pos in range(p0, p1):
            assert set(bp.neighborhood(osk.a, osk.b, osk.M, 8, orbit[pos])) <= set(blocks)
    assert covered == list(range(1024))
    assert math.isclose(D.halo_overhead(1024, 8, 8), 7 / 128)


class _OracleRanks:
    """Test double for the CUDA range apply: uses only A_local (stacked blocks)."""

    def __init__(self, osk):
        self.osk = osk
        self.M, self.B_r = osk.M, osk.B_r
        self._orbit = bp.orbit(osk.a, osk.b, osk.M)

    def orbit(self):
        return self._orbit

    def apply_range(self, p0, p1, A_local):
        sk = self.osk
        A = A_local.numpy().astype(np.float64)
        Y = np.zeros(((p1 - p0) * sk.B_r, A.shape[1]))
        for i in range(p0, p1):
            g = self._orbit[i % sk.M]
            for ell in range(1, sk.kappa + 1):
                blk = A[(i - p0 + ell - 1) * sk.B_c:(i - p0 + ell) * sk.B_c]
                for u in range(sk.B_c):
                    for j in range(sk.s):
                        r, sg = bp.pattern(sk, g, ell, u, j)
                        Y[(i - p0) * sk.B_r + r] += sg * blk[u]
        return torch.from_numpy(Y / math.sqrt(sk.kappa * sk.s))


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        osk = oracle.make_sketch(8, 32, 128, 2, 2, 1234)  # tiny config
        sk = _OracleRanks(osk)
        rng = np.random.default_rng(7)
        A = rng.standard_normal((osk.d, 5))
        p0, p1 = D.orbit_shard(osk.M, world, rank)
        blocks = D.input_blocks(sk.orbit(), p0, p1, osk.kappa)
        A_local = torch.from_numpy(np.concatenate([A[h * osk.B_c:(h + 1) * osk.B_c] for h in blocks]))
        Y = D.block_sharded_apply(sk, A_local, apply_range=sk.apply_range)
        ref = oracle.apply(osk, A)
        out_q.put((rank, float(np.abs(Y.numpy() - ref).max())))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_block_sharded_apply_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for rank, err in res:
        assert err < 1e-12, (rank, err)


class _FakeSymmetric:
    """Emulates torch symmetric memory for the CPU test: 'peer pointers' are rank ids; the stores a
    rank's kernel would make into every peer's buffer are replayed at the barrier through gloo."""

    def __init__(self, sk):
        self.sk = sk
        self.pending = []

    def rendezvous(self, shape, device, group):
        self.world = dist.get_world_size(group)
        self.buf = torch.full(shape, float("nan"), dtype=torch.float64)
        return self.buf, list(range(self.world)), 0, self.barrier

    def apply_range(self, p0, p1, A_local, dst, mc, row0):
        assert tuple(dst) == tuple(range(self.world)) and mc == 0
        self.pending.append((row0, self.sk.apply_range(p0, p1, A_local)))

    def barrier(self):
        got = [None] * self.world
        dist.all_gather_object(got, self.pending)
        for lst in got:
            for row0, Y in lst:
                self.buf[row0:row0 + Y.shape[0]] = Y


def _worker_fused(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        osk = oracle.make_sketch(8, 32, 128, 2, 2, 1234)
        sk = _OracleRanks(osk)
        rng = np.random.default_rng(8)
        A = rng.standard_normal((osk.d, 5))
        p0, p1 = D.orbit_shard(osk.M, world, rank)
        blocks = D.input_blocks(sk.orbit(), p0, p1, osk.kappa)
        A_local = torch.from_numpy(np.concatenate([A[h * osk.B_c:(h + 1) * osk.B_c] for h in blocks]))
        fake = _FakeSymmetric(sk)
        Y = D.block_sharded_apply_fused(sk, A_local, rendezvous=fake.rendezvous, apply_range=fake.apply_range)
        ref = oracle.apply(osk, A)
        out_q.put((rank, float(np.abs(Y.numpy() - ref).max())))
    finally:
        dist.destroy_process_group()


def test_block_sharded_apply_fused_gloo():
    """Host logic of the fused (epilogue-broadcast) block sharding: destination rows p0·B_r.. of every
    rank's orbit-ordered buffer, one barrier, orbit→g permutation — world 2 on CPU."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_fused, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for rank, err in res:
        assert err < 1e-12, (rank, err)

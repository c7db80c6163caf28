"""Multi-GPU partitioner for Y = S·A.

Two shardings, one process per GPU (torch.distributed, NCCL over NVLink/NVSwitch):

* column sharding — rank r applies the same S to its own column range; no collective.
* orbit block sharding — for very large d.  Ordering blocks along the wiring orbit
  g_pos = f^pos(0) makes every output block's neighbourhood a window of the
  next κ positions, so rank r, owning output positions [p0, p1), needs only input positions
  p0+1 .. p1+κ-1: 1/P of A plus a κ-1 block halo.  It runs bps_apply_orbit_range on its
  stacked blocks; one all_gather_into_tensor assembles Y in orbit order and a row-block
  permutation restores g order.

The per-rank compute is injectable (`apply_range`) so the partitioning and collective logic
can be tested on CPU with gloo; the production default calls the CUDA library.
"""

from __future__ import annotations

from typing import Callable, Sequence


def column_shard(n: int, world: int, rank: int, align: int = 128) -> tuple[int, int]:
    """Contiguous column range of `rank`, boundaries multiples of `align` (tile width)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    units = -(-n // align)
    u0 = units * rank // world
    u1 = units * (rank + 1) // world
    return min(n, u0 * align), min(n, u1 * align)


def orbit_shard(M: int, world: int, rank: int) -> tuple[int, int]:
    """Output orbit positions [p0, p1) owned by `rank` (balanced, contiguous)."""
    if world < 1 or not (0 <= rank < world) or world > M:
        raise ValueError("need 1 <= world <= M and 0 <= rank < world")
    return M * rank // world, M * (rank + 1) // world


def halo_positions(p0: int, p1: int, kappa: int) -> list[int]:
    """Input orbit positions a rank owning outputs [p0, p1) reads: p0+1 .. p1+κ-1."""
    return list(range(p0 + 1, p1 + kappa))


def input_blocks(orbit: Sequence[int], p0: int, p1: int, kappa: int) -> list[int]:
    """Input block ids g (rows g·B_c..) in the stacking order bps_apply_orbit_range expects."""
    M = len(orbit)
    return [orbit[p % M] for p in halo_positions(p0, p1, kappa)]


def halo_overhead(M: int, world: int, kappa: int) -> float:
    """Fraction of extra input rows read because of the κ-1 block halo."""
    per = M / world
    return (per + kappa - 1) / per - 1.0


def gather_orbit_to_g(Y_orbit, orbit: Sequence[int], B_r: int):
    """Reorder row blocks from orbit order (block i = output g_{i}) to g order."""
    import torch

    M = len(orbit)
    pos_of_g = [0] * M
    for pos, g in enumerate(orbit):
        pos_of_g[g] = pos
    rows = torch.arange(B_r, device=Y_orbit.device)
    idx = torch.cat([pos_of_g[g] * B_r + rows for g in range(M)])
    return Y_orbit.index_select(0, idx)


def block_sharded_apply(sk, A_local, group=None, apply_range: Callable | None = None, out=None):
    """Orbit block-sharded Y = S·A across the ranks of `group`.

    A_local: this rank's stacked input blocks (input_blocks(...) order), n columns.
    Returns the full k×n Y (g order) on every rank.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    M, B_r = sk.M, sk.B_r
    if M % world:
        raise ValueError("block sharding needs M % world == 0 (equal all-gather chunks)")
    p0, p1 = orbit_shard(M, world, rank)
    if apply_range is None:
        Y_loc = sk.apply_orbit_range(p0, p1, A_local)
    else:
        Y_loc = apply_range(p0, p1, A_local)
    Y_loc = Y_loc.contiguous()
    Y_orbit = torch.empty((M * B_r, Y_loc.shape[1]), dtype=Y_loc.dtype, device=Y_loc.device)
    dist.all_gather_into_tensor(Y_orbit, Y_loc, group=group)
    Y = gather_orbit_to_g(Y_orbit, sk.orbit() if hasattr(sk, "orbit") else sk["orbit"], B_r)
    if out is not None:
        out.copy_(Y)
        return out
    return Y

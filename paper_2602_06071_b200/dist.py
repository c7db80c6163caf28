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


def symmetric_rendezvous(shape, device, group=None):
    """Allocate a symmetric fp32 buffer on every rank of `group` (torch symmetric memory) and return
    (buffer, peer pointers (one per rank, valid in this process), multicast address or 0, barrier)."""
    import torch
    import torch.distributed._symmetric_memory as symm_mem

    key = (tuple(shape), str(device), group if isinstance(group, str) else id(group))
    if key in _SYMM:  # one symmetric buffer per (shape, device, group), reused across calls
        return _SYMM[key]
    buf = symm_mem.empty(shape, dtype=torch.float32, device=device)
    hdl = symm_mem.rendezvous(buf, group if group is not None else _default_group_name())
    ptrs = [int(p) for p in hdl.buffer_ptrs]
    mc = int(getattr(hdl, "multicast_ptr", 0) or 0)
    _SYMM[key] = (buf, ptrs, mc, lambda: hdl.barrier(channel=0))
    return _SYMM[key]


_SYMM: dict = {}


def _default_group_name():
    import torch.distributed as dist

    return dist.group.WORLD.group_name


def block_sharded_apply_fused(sk, A_local, group=None, rendezvous: Callable | None = None,
                              apply_range: Callable | None = None, multicast: bool = True, variant: str = "auto"):
    """Orbit block-sharded Y = S·A with the all-gather fused into the kernel epilogue (SURVEY §8(e)
    B200-native step): rank r's kernel stores each finished output tile of its orbit
    positions [p0, p1) straight into EVERY rank's symmetric orbit-ordered Y buffer — one multimem.st
    through the NVLS multicast address when the symmetric-memory handle exposes one, else one store
    per peer pointer over NVLink (bps_apply_orbit_range_bcast) — then one cross-GPU barrier; no
    separate collective pass.  Returns the full k×n Y (g order) on every rank, bitwise equal to
    block_sharded_apply and to the 1-GPU apply (R19).

    rendezvous(shape, device, group) -> (buffer, peer_ptrs, mc_ptr, barrier) and
    apply_range(p0, p1, A_local, dst_ptrs, mc_ptr, dst_row0) are injectable for the CPU (gloo) tests.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    M, B_r = sk.M, sk.B_r
    p0, p1 = orbit_shard(M, world, rank)
    n = A_local.shape[1]
    rv = rendezvous or symmetric_rendezvous
    Y_orbit, ptrs, mc, barrier = rv((M * B_r, n), A_local.device, group)
    if not (multicast and mc):
        mc = 0
    dst = () if mc else tuple(ptrs)
    if apply_range is None:
        sk.apply_orbit_range(p0, p1, A_local, variant=variant, dst=dst, mc_ptr=mc, dst_ld=Y_orbit.stride(0),
                             dst_row0=p0 * B_r)
    else:
        apply_range(p0, p1, A_local, dst, mc, p0 * B_r)
    barrier()  # every rank's stores have landed in every buffer
    orbit = sk.orbit() if hasattr(sk, "orbit") else sk["orbit"]
    return gather_orbit_to_g(Y_orbit, orbit, B_r)

"""Multi-GPU plumbing: one process per GPU, NCCL communicator bootstrapped over
torch.distributed, and the row/tile partitions the library uses.

The partitions are restated here in Python (identical arithmetic to
csrc/gpk_api.cu: gpk_shard_rows, quad_forms_dev's tile split and
grad_kernel's triangle enumeration) so the decomposition can be tested on CPU
with a gloo process group (tests/test_multi_gloo.py)."""
from __future__ import annotations

import ctypes as C
import math

from . import _lib
from ._lib import check


def comm_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    check(_lib.load().gpk_comm_unique_id(buf))
    return bytes(buf)


def init_comm_from_torch(ctx, group=None):
    """Rank 0 creates the NCCL id; torch.distributed broadcasts it; every rank joins."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    obj = [comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.init_comm(obj[0], world, rank)
    return world, rank


def shard_stride(n: int, nranks: int) -> int:
    """Rows per rank, rounded up to whole 32-row operator chunks (gpk_shard_rows)."""
    return ((n + nranks - 1) // nranks + 31) // 32 * 32


def shard_rows(n: int, nranks: int, rank: int):
    """[row0, row1) owned by `rank` (gpk_shard_rows)."""
    S = shard_stride(n, nranks)
    return min(n, rank * S), min(n, (rank + 1) * S)


def shard_rows_c(n: int, nranks: int, rank: int):
    """The library's own gpk_shard_rows (callable without a GPU)."""
    r0, r1 = C.c_int(), C.c_int()
    check(_lib.load().gpk_shard_rows(n, nranks, rank, C.byref(r0), C.byref(r1)))
    return r0.value, r1.value


TILE = 64  # grad_kernel tile edge


def grad_tile_range(n: int, nranks: int, rank: int, symmetric: bool = True):
    """Global tile-index range of the gradient pass owned by `rank` (quad_forms_dev)."""
    T = (n + TILE - 1) // TILE
    ntiles = T * (T + 1) // 2 if symmetric else T * T
    return ntiles * rank // nranks, ntiles * (rank + 1) // nranks


def tile_coords(L: int, n: int, symmetric: bool = True):
    """(ti, tc) of linear tile L: row-major upper triangle when symmetric (grad_kernel tile_coords)."""
    T = (n + TILE - 1) // TILE
    if not symmetric:
        return L // T, L % T
    b = 2.0 * T + 1.0
    r = int((b - math.sqrt(b * b - 8.0 * L)) / 2.0)
    r = max(0, min(r, T - 1))

    def off(rr):
        return rr * T - rr * (rr - 1) // 2

    while r > 0 and off(r) > L:
        r -= 1
    while r + 1 < T and off(r + 1) <= L:
        r += 1
    return r, r + (L - off(r))

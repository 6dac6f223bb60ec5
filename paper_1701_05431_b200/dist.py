"""Host-side logic of the multi-process (one GPU per rank) path.

The data path (boundary rows, halo rows, the max-all-reduce of the CFL speed)
runs inside libfv2d over NCCL; this module holds what the host does around it:
the y-slab partition (ny % P == 0), the neighbour map (R10: +y =
north = rank+1, periodic ring), broadcasting the NCCL unique id, and the
max-over-ranks reductions bench.py uses for timing.  `exchange_halo_rows`
is the same send/recv protocol the library posts to NCCL (ncclGroupStart;
Send(bottom -> south); Recv(north ghost <- north); Send(top -> north);
Recv(south ghost <- south); ncclGroupEnd), written with torch.distributed
point-to-point calls so the protocol itself can be tested with the gloo
backend on CPU (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import numpy as np


def slab_rows(rank: int, world: int, ny: int) -> tuple[int, int]:
    """Rows [j0, j1) of rank's y-slab."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    if ny % world:
        raise ValueError(f"ny={ny} is not divisible by {world} ranks")
    h = ny // world
    return rank * h, (rank + 1) * h


def neighbours(rank: int, world: int, periodic: bool = True):
    """(south, north) neighbour ranks; None at a non-periodic physical boundary."""
    south = (rank - 1) % world if (rank > 0 or periodic) else None
    north = (rank + 1) % world if (rank < world - 1 or periodic) else None
    return south, north


def block_of(rank: int, px: int, py: int, nx: int, ny: int) -> tuple[int, int, int, int]:
    """(j0, j1, i0, i1) of rank's 2-D block: the ranks form a px x py grid,
    rank = ry*px + rx (fv2d.h nranks_x; the paper's NPartX x NPartY)."""
    if px < 1 or py < 1 or not (0 <= rank < px * py):
        raise ValueError(f"bad rank {rank} of {px}x{py}")
    if nx % px or ny % py or nx // px < 2:
        raise ValueError(f"{nx}x{ny} cells do not split into {px}x{py} blocks of >= 2 columns")
    rx, ry = rank % px, rank // px
    w, h = nx // px, ny // py
    return ry * h, (ry + 1) * h, rx * w, (rx + 1) * w


def block_neighbours(rank: int, px: int, py: int, periodic_x: bool = True, periodic_y: bool = True):
    """(south, north, west, east) neighbour ranks of a 2-D block; None at a
    non-periodic physical boundary (the four overlaps of P:359-374)."""
    rx, ry = rank % px, rank // px
    at = lambda x, y: (y % py) * px + (x % px)  # noqa: E731
    south = at(rx, ry - 1) if (ry > 0 or periodic_y) else None
    north = at(rx, ry + 1) if (ry < py - 1 or periodic_y) else None
    west = at(rx - 1, ry) if (rx > 0 or periodic_x) else None
    east = at(rx + 1, ry) if (rx < px - 1 or periodic_x) else None
    return south, north, west, east


def exchange_halo_2d(block: np.ndarray, rank: int, px: int, py: int, periodic_x: bool = True,
                     periodic_y: bool = True):
    """The library's NCCL group for 2-D blocks, with torch.distributed p2p:
    rows as exchange_halo_rows, then columns in the same pattern (Send(west
    column -> west); Recv(east ghost <- east); Send(east column -> east);
    Recv(west ghost <- west)), all in one batch.  Returns (south, north, west,
    east) ghost lines (None at a physical boundary)."""
    import torch
    import torch.distributed as dist
    s, n, w, e = block_neighbours(rank, px, py, periodic_x, periodic_y)
    lines = {"s": np.ascontiguousarray(block[0]), "n": np.ascontiguousarray(block[-1]),
             "w": np.ascontiguousarray(block[:, 0]), "e": np.ascontiguousarray(block[:, -1])}
    recv = {}
    ops = []
    for lo, hi, plo, phi in (("s", "n", s, n), ("w", "e", w, e)):
        if plo == rank and phi == rank:  # one block along this axis: its own neighbour
            recv[hi], recv[lo] = torch.from_numpy(lines[lo].copy()), torch.from_numpy(lines[hi].copy())
            continue
        if plo is not None:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(lines[lo]), plo))
        if phi is not None:
            recv[hi] = torch.empty(lines[hi].shape, dtype=torch.float64)
            ops.append(dist.P2POp(dist.irecv, recv[hi], phi))
        if phi is not None:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(lines[hi]), phi))
        if plo is not None:
            recv[lo] = torch.empty(lines[lo].shape, dtype=torch.float64)
            ops.append(dist.P2POp(dist.irecv, recv[lo], plo))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return tuple(None if k not in recv else recv[k].numpy() for k in ("s", "n", "w", "e"))


def broadcast_bytes(payload: bytes | None, src: int = 0) -> bytes:
    """Broadcast a small byte string (the 128-byte NCCL unique id) from src."""
    import torch.distributed as dist
    obj = [payload]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def max_over_ranks(values, device="cpu"):
    """Element-wise max over ranks (timings are reported as the max, never the mean)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def exchange_halo_rows(bottom_row: np.ndarray, top_row: np.ndarray, rank: int, world: int, periodic: bool = True):
    """Send my bottom row south and my top row north; return (south_ghost,
    north_ghost) received from the neighbours (None at a physical boundary).
    Posting order per peer matches the library's NCCL group, so with two ranks
    (both neighbours are the same peer) the FIFO matching still pairs each row
    with the right ghost."""
    import torch
    import torch.distributed as dist
    south, north = neighbours(rank, world, periodic)
    ops = []
    recv_n = recv_s = None
    if south is not None:
        ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(bottom_row)), south))
    if north is not None:
        recv_n = torch.empty(top_row.shape, dtype=torch.float64)
        ops.append(dist.P2POp(dist.irecv, recv_n, north))
    if north is not None:
        ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(top_row)), north))
    if south is not None:
        recv_s = torch.empty(bottom_row.shape, dtype=torch.float64)
        ops.append(dist.P2POp(dist.irecv, recv_s, south))
    if world == 1:
        # self exchange (the library's FV2D_FLAG_NCCL_LOOPBACK case)
        return (top_row.copy() if south is not None else None, bottom_row.copy() if north is not None else None)
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    return (None if recv_s is None else recv_s.numpy(), None if recv_n is None else recv_n.numpy())

"""Multi-GPU execution of the hot path.

Two decompositions:

* **Independent pairs (config 4)** -- replicas: every rank registers its own pairs;
  no data-path collective (see `bench.py --gpus N`).
* **z-slabs of one large pair (config 5)** -- every rank holds the template, the
  reference terms of its slab and the full (small) deformation grid; it evaluates
  the fused NGF pipeline only for image planes [zlo, zhi).  Because G^T, the warp
  Jacobian transpose and P^T are linear, the ring planes at a slab boundary carry
  exactly that slab's contributions (the same argument the fused kernel uses at its
  own chunk boundaries), so the objective gradient is the SUM of the slab partials.
  Per evaluation (default `exchange="planes"`): each rank's partial is non-zero only on
  the deformation planes its slab touches (its *window*); the planes are partitioned
  among the ranks (*owned* ranges), every rank sends the window planes owned by other
  ranks to their owners (point-to-point, a plane or two per neighbour), each owner sums
  the contributions of its planes in rank order (deterministic for a given G), and an
  all-gather of the owned planes gives every rank the full grad D -- half the bytes of
  an all-reduce of the 3M vector.  `exchange="allreduce"` keeps the simple all-reduce.
  D is all-reduced as a scalar; then every rank adds the curvature term identically
  and runs the same (replicated) L-BFGS step.

The collective logic lives in `SlabObjective`, independent of where the slab partial
comes from: on GPUs it is the sm_100a level (`DeviceSlab`) with NCCL; the CPU tests
plug an oracle slab evaluator and the gloo backend into the same class.
"""

from __future__ import annotations

import math

import numpy as np

from . import _device as dev
from ._lib import check, lib

__all__ = ["slab_ranges", "slab_plane_layout", "SlabObjective", "DeviceSlab"]


def slab_ranges(nz: int, nd_z: int, world: int):
    """Contiguous image z-ranges, one per rank, cut at deformation-cell boundaries
    when the grid ratio is an integer (so slab windows overlap by the minimum)."""
    if world < 1 or world > nz:
        raise ValueError(f"cannot split {nz} planes over {world} ranks")
    ratio = nz // nd_z if nd_z > 0 and nz % nd_z == 0 else 1
    units = nz // ratio
    cuts = [round(r * units / world) * ratio for r in range(world + 1)]
    cuts[-1] = nz
    out = [(cuts[r], cuts[r + 1]) for r in range(world)]
    if any(lo >= hi for lo, hi in out):
        raise ValueError(f"{world} ranks leave an empty slab for nz={nz}")
    return out


def _i0(z: int, oz: float, hz: float, odz: float, hdz: float, ndz: int) -> int:
    # transfer.py:54-63 (the z-axis index map)
    if ndz < 2:
        return 0
    return min(max(int(math.floor((oz + z * hz - odz) / hdz)), 0), ndz - 2)


def slab_plane_layout(image_grid, def_grid, slabs):
    """Per rank: the deformation planes its slab partial can touch (window, inclusive,
    with a one-plane margin) and the planes it owns (a partition of [0, ndz)).
    `image_grid` / `def_grid` need .dims, .spacing, .origin."""
    nz, hz, oz = image_grid.dims[2], image_grid.spacing[2], image_grid.origin[2]
    ndz, hdz, odz = def_grid.dims[2], def_grid.spacing[2], def_grid.origin[2]
    windows, cuts = [], []
    for zlo, zhi in slabs:
        # image planes [zlo - 1, zhi] carry the slab's G^T / J^T contributions; one more
        # each side as margin (planes of zeros are harmless)
        lo = _i0(max(zlo - 2, 0), oz, hz, odz, hdz, ndz)
        hi = min(_i0(min(zhi + 1, nz - 1), oz, hz, odz, hdz, ndz) + 1, ndz - 1)
        windows.append((lo, hi))
        cuts.append(_i0(zlo, oz, hz, odz, hdz, ndz) if zlo > 0 else 0)
    cuts.append(ndz)
    for r in range(1, len(cuts)):
        cuts[r] = min(max(cuts[r], cuts[r - 1]), ndz)
    owned = [(cuts[r], cuts[r + 1]) for r in range(len(slabs))]
    return windows, owned


class DeviceSlab:
    """Slab partial of a device level (`DeviceLevel` restricted to [zlo, zhi))."""

    def __init__(self, level, zlo: int, zhi: int):
        check(lib().ngf_level_set_zrange(level.handle, int(zlo), int(zhi)), "ngf_level_set_zrange")
        self.level = level
        self.zlo, self.zhi = zlo, zhi
        self.image_grid, self.def_grid = level.image_grid, level.def_grid

    def partial(self, x, grad, scal):
        """grad <- grad D_slab, scal[1] <- D_slab (device, no sync)."""
        check(lib().ngf_level_eval(self.level.handle, dev.ptr(x), dev.ptr(grad), dev.ptr(scal), 2,
                                   dev.stream()), "ngf_level_eval(slab)")

    def finish(self, x, grad, scal):
        """grad += alpha grad S; scal <- (J, D, S) with D = scal[1] (already summed)."""
        check(lib().ngf_level_add_curvature(self.level.handle, dev.ptr(x), dev.ptr(grad), dev.ptr(scal),
                                            dev.stream()), "ngf_level_add_curvature")


class SlabObjective:
    """Objective over a z-slab decomposition; identical results on every rank.

    `local` provides partial(x, grad, scal) and finish(x, grad, scal) on tensors and the
    attributes zlo, zhi, image_grid, def_grid; `group` is a torch.distributed process
    group (NCCL for GPUs, gloo in CPU tests).
    """

    def __init__(self, local, group=None, exchange: str = "planes"):
        if exchange not in ("planes", "allreduce"):
            raise ValueError(f"unknown exchange {exchange!r}")
        self.local = local
        self.group = group
        self.exchange = exchange
        self.evals = 0
        self._layout = None

    def _plan(self):
        import torch.distributed as dist

        if self._layout is None:
            ws = dist.get_world_size(self.group)
            mine = (int(self.local.zlo), int(self.local.zhi))
            slabs = [None] * ws
            dist.all_gather_object(slabs, mine, group=self.group)
            self._layout = slab_plane_layout(self.local.image_grid, self.local.def_grid, slabs)
        return self._layout

    def _exchange_planes(self, grad):
        import torch
        import torch.distributed as dist

        ws = dist.get_world_size(self.group)
        rank = dist.get_rank(self.group)
        windows, owned = self._plan()
        nd = self.local.def_grid.dims
        g = grad.view(3, nd[2], nd[1] * nd[0])

        def overlap(q, r):
            lo = max(windows[q][0], owned[r][0])
            hi = min(windows[q][1] + 1, owned[r][1])
            return (lo, hi) if lo < hi else None

        # window planes owned by other ranks go to their owners
        ops, recv = [], {}
        for r in range(ws):
            if r == rank:
                continue
            ov = overlap(rank, r)
            if ov:
                ops.append(dist.P2POp(dist.isend, g[:, ov[0]:ov[1]].contiguous(), r, self.group))
            ov = overlap(r, rank)
            if ov:
                buf = torch.empty((3, ov[1] - ov[0], g.shape[2]), dtype=g.dtype, device=g.device)
                recv[r] = (ov, buf)
                ops.append(dist.P2POp(dist.irecv, buf, r, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        # owner sum in rank order (own contribution at its rank position)
        olo, ohi = owned[rank]
        acc = torch.zeros((3, ohi - olo, g.shape[2]), dtype=g.dtype, device=g.device)
        for q in range(ws):
            ov = overlap(q, rank)
            if not ov:
                continue
            part = g[:, ov[0]:ov[1]] if q == rank else recv[q][1]
            acc[:, ov[0] - olo:ov[1] - olo] += part
        # all-gather of the owned planes (padded to the largest owned range)
        width = max(hi - lo for lo, hi in owned)
        mine = torch.zeros((3, width, g.shape[2]), dtype=g.dtype, device=g.device)
        mine[:, :ohi - olo] = acc
        blocks = [torch.empty_like(mine) for _ in range(ws)]
        dist.all_gather(blocks, mine, group=self.group)
        for q, (lo, hi) in enumerate(owned):
            g[:, lo:hi] = blocks[q][:, :hi - lo]

    def eval_device(self, x, grad, scal):
        import torch.distributed as dist

        self.evals += 1
        self.local.partial(x, grad, scal)
        if dist.is_initialized():
            if self.exchange == "planes":
                self._exchange_planes(grad)
            else:
                dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=self.group)
            d = scal[1:2].clone()
            dist.all_reduce(d, op=dist.ReduceOp.SUM, group=self.group)
            scal[1:2].copy_(d)
        self.local.finish(x, grad, scal)
        return scal


def weak_scaling_pairs(total_pairs: int, world: int, rank: int):
    """Config 4: which of `total_pairs` independent pairs this rank registers."""
    per = math.ceil(total_pairs / world)
    return list(range(rank * per, min(total_pairs, (rank + 1) * per)))


def as_numpy(t):
    return t.detach().cpu().numpy() if dev.is_tensor(t) else np.asarray(t)

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
  Per evaluation: one all-reduce of grad D (3M values) and of D, then every rank adds
  the curvature term identically and runs the same (replicated) L-BFGS step.

The collective logic lives in `SlabObjective`, independent of where the slab partial
comes from: on GPUs it is the sm_100a level (`DeviceSlab`) with NCCL; the CPU tests
plug an oracle slab evaluator and the gloo backend into the same class.
"""

from __future__ import annotations

import math

import numpy as np

from . import _device as dev
from ._lib import check, lib

__all__ = ["slab_ranges", "SlabObjective", "DeviceSlab"]


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


class DeviceSlab:
    """Slab partial of a device level (`DeviceLevel` restricted to [zlo, zhi))."""

    def __init__(self, level, zlo: int, zhi: int):
        check(lib().ngf_level_set_zrange(level.handle, int(zlo), int(zhi)), "ngf_level_set_zrange")
        self.level = level
        self.zlo, self.zhi = zlo, zhi

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

    `local` provides partial(x, grad, scal) and finish(x, grad, scal) on tensors;
    `group` is a torch.distributed process group (NCCL for GPUs, gloo in CPU tests).
    """

    def __init__(self, local, group=None):
        self.local = local
        self.group = group
        self.evals = 0

    def eval_device(self, x, grad, scal):
        import torch.distributed as dist

        self.evals += 1
        self.local.partial(x, grad, scal)
        if dist.is_initialized():
            # fixed-size reductions; NCCL's ring order is fixed for a given topology
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

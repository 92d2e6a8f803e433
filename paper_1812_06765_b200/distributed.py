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

__all__ = ["slab_ranges", "slab_plane_layout", "combine_slab_partials", "SlabObjective", "LocalSlabGroup",
           "DeviceSlab", "register_slab"]


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


def _overlap(windows, owned, q, r):
    lo = max(windows[q][0], owned[r][0])
    hi = min(windows[q][1] + 1, owned[r][1])
    return (lo, hi) if lo < hi else None


def combine_slab_partials(partials, windows, owned):
    """grad D from the slab partials exactly as the distributed plane exchange forms it:
    for every owner r (in rank order), its planes are the sum, in rank order q = 0, 1, ...,
    of the contributions of the slabs whose windows overlap them (zeros where none does).
    `partials` are torch tensors (3, ndz, rest), one per rank.  One-process reference of
    SlabObjective's exchange (bit-identical for the same partials)."""
    import torch

    out = torch.zeros_like(partials[0])
    for r in range(len(owned)):
        olo, ohi = owned[r]
        acc = torch.zeros_like(out[:, olo:ohi])
        for q in range(len(partials)):
            ov = _overlap(windows, owned, q, r)
            if ov:
                acc[:, ov[0] - olo:ov[1] - olo] += partials[q][:, ov[0]:ov[1]]
        out[:, olo:ohi] = acc
    return out


def ordered_sum(values):
    """Sum of per-rank scalars in rank order (the distributed D)."""
    acc = 0.0
    for v in values:
        acc = acc + float(v)
    return acc


class DeviceSlab:
    """Slab partial of a device level (`DeviceLevel` restricted to [zlo, zhi))."""

    def __init__(self, level, zlo: int, zhi: int, restrict: bool = True):
        if restrict:
            check(lib().ngf_level_set_zrange(level.handle, int(zlo), int(zhi)), "ngf_level_set_zrange")
        self.level = level
        self.zlo, self.zhi = zlo, zhi
        self.image_grid, self.def_grid = level.image_grid, level.def_grid

    @classmethod
    def create(cls, image_grid, def_grid, T_dev, R_dev, params, alpha: float, zlo: int, zhi: int):
        """A slab level whose reference terms are computed on planes [zlo, zhi) only
        (ngf_level_create_zslab): the template and R are replicated, nothing else is."""
        import ctypes

        from ._lib import dtype_code, ngf_grid
        from .objective import DeviceLevel

        lvl = DeviceLevel.__new__(DeviceLevel)
        lvl.image_grid, lvl.def_grid = image_grid, def_grid
        lvl.dtype = T_dev.dtype
        lvl.T, lvl._R = T_dev, R_dev
        lvl.alpha = float(alpha)
        h = ctypes.c_void_p()
        ig, dg = ngf_grid(image_grid), ngf_grid(def_grid)
        check(lib().ngf_level_create_zslab(ctypes.byref(ig), ctypes.byref(dg), dtype_code(T_dev.dtype),
                                           dev.ptr(T_dev), dev.ptr(R_dev), float(params.tau), float(params.rho),
                                           lvl.alpha, int(zlo), int(zhi), dev.stream(), ctypes.byref(h)),
              "ngf_level_create_zslab")
        lvl.handle = h
        lvl.n = 3 * def_grid.num_points
        lvl.scalars = dev.zeros((3,), "float64")
        return cls(lvl, zlo, zhi, restrict=False)

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
            return _overlap(windows, owned, q, r)

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
        import torch
        import torch.distributed as dist

        self.evals += 1
        self.local.partial(x, grad, scal)
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            if self.exchange == "planes":
                self._exchange_planes(grad)
            else:
                dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=self.group)
            # D: the slab values gathered and summed in rank order (deterministic for a
            # given world size, whatever order the backend's all-reduce would use)
            d = scal[1:2].clone()
            ds = [torch.empty_like(d) for _ in range(dist.get_world_size(self.group))]
            dist.all_gather(ds, d, group=self.group)
            scal[1] = ordered_sum(v.item() for v in ds)
        self.local.finish(x, grad, scal)
        return scal

    def __call__(self, x):
        """The reference's objective contract, numpy in -> (J, numpy grad) out
        (objective.py:54-60), identical on every rank."""
        return _numpy_call(self, _is_device(self.local), x)


class LocalSlabGroup:
    """All slabs of a decomposition evaluated in ONE process and combined exactly like
    SlabObjective over a process group (plane exchange in rank order, D summed in rank
    order): the single-process reference a distributed run is compared against
    bit-for-bit, and a way to run the config-5 decomposition on one device."""

    def __init__(self, slabs):
        self.slabs = list(slabs)
        self.evals = 0
        first = self.slabs[0]
        self.image_grid, self.def_grid = first.image_grid, first.def_grid
        self.layout = slab_plane_layout(first.image_grid, first.def_grid,
                                        [(int(s.zlo), int(s.zhi)) for s in self.slabs])

    def eval_device(self, x, grad, scal):
        import torch

        self.evals += 1
        nd = self.def_grid.dims
        parts, ds = [], []
        for s in self.slabs:
            g = torch.empty_like(grad)
            sc = torch.zeros_like(scal)
            s.partial(x, g, sc)
            parts.append(g.view(3, nd[2], nd[1] * nd[0]))
            ds.append(float(sc[1].item()))
        windows, owned = self.layout
        grad.view(3, nd[2], nd[1] * nd[0]).copy_(combine_slab_partials(parts, windows, owned))
        scal[1] = ordered_sum(ds)
        self.slabs[0].finish(x, grad, scal)
        return scal

    def __call__(self, x):
        return _numpy_call(self, _is_device(self.slabs[0]), x)


def _is_device(slab) -> bool:
    return hasattr(getattr(slab, "level", None), "handle")


def _numpy_call(obj, on_gpu: bool, x):
    import torch

    xa = np.asarray(x)
    if not np.all(np.isfinite(xa)):
        # overflowed line-search trial point; force a backtrack (objective.py:55-57)
        return float("inf"), np.zeros_like(xa)
    xt = torch.from_numpy(np.ascontiguousarray(xa).reshape(-1).copy())
    if on_gpu:
        xt = xt.cuda()
    g = torch.empty_like(xt)
    sc = torch.zeros(3, dtype=torch.float64, device=xt.device)
    obj.eval_device(xt, g, sc)
    return float(sc[0].item()), g.cpu().numpy().reshape(xa.shape)


def weak_scaling_pairs(total_pairs: int, world: int, rank: int):
    """Config 4: which of `total_pairs` independent pairs this rank registers."""
    per = math.ceil(total_pairs / world)
    return list(range(rank * per, min(total_pairs, (rank + 1) * per)))


def as_numpy(t):
    return t.detach().cpu().numpy() if dev.is_tensor(t) else np.asarray(t)


def register_slab(R, T, cfg=None, group=None, emulate_world: int | None = None):
    """Config 5: ONE registration (multilevel.py:179-247) with every level z-slab
    decomposed over the ranks of `group`.

    Each rank holds the template and R (replicated, read-only), builds both pyramids, and
    per level creates a slab level whose reference terms cover its own planes only
    (`DeviceSlab.create`); `SlabObjective` combines the slab partials (plane exchange +
    D in rank order), and the L-BFGS state is replicated: every rank runs the same
    `lbfgs_minimize` on identical (J, grad J), so the ranks stay in lock-step with no
    further communication.  With `emulate_world=G` and no process group, the G slabs of
    each level are evaluated in this process (`LocalSlabGroup`) -- the bit-for-bit
    single-process reference of a G-rank run.  Returns (DeformationField, report)."""
    import time

    import torch.distributed as dist

    from .geometry import DeformationField, identity_field_array, precision_dtype
    from .lbfgs import lbfgs_minimize
    from .multilevel import (LevelReport, MultilevelConfig, RegistrationReport, _coarser, _downsample_dev,
                             _prolong_dev, deformation_grid_for, num_auto_levels)

    cfg = cfg or MultilevelConfig()
    if R.grid != T.grid:
        from ._lib import GridError
        raise GridError("reference and template must share one grid; resample the template first")
    distributed = emulate_world is None and dist.is_initialized()
    world = dist.get_world_size(group) if distributed else (emulate_world or 1)
    rank = dist.get_rank(group) if distributed else 0
    t_start = time.perf_counter()
    dtype = precision_dtype(cfg.precision)
    levels = cfg.num_levels or num_auto_levels(R.grid.dims, cfg.coarsest_min_dim)
    np_out = not dev.is_tensor(R.values)
    Rv = R.values.astype(dtype, copy=False) if np_out else R.values
    Tv = T.values.astype(dtype, copy=False) if not dev.is_tensor(T.values) else T.values
    pyr = [(dev.to_device(Rv, dtype), dev.to_device(Tv, dtype), R.grid)]
    for _ in range(levels - 1):
        r_, t_, g = pyr[-1]
        ng = _coarser(g)
        if ng.dims == g.dims:
            raise ValueError(f"cannot build {levels} levels from dims {R.grid.dims}")
        pyr.append((_downsample_dev(r_, g), _downsample_dev(t_, g), ng))
    pyr.reverse()
    report = RegistrationReport(seconds_pyramid=time.perf_counter() - t_start)
    y = prev = None
    for lvl, (R_l, T_l, gi) in enumerate(pyr):
        t0 = time.perf_counter()
        gd = deformation_grid_for(gi, cfg.grid_ratio)
        slabs = slab_ranges(gi.dims[2], gd.dims[2], world)
        if distributed:
            zlo, zhi = slabs[rank]
            obj = SlabObjective(DeviceSlab.create(gi, gd, T_l, R_l, cfg.ngf, cfg.alpha, zlo, zhi), group)
        else:
            obj = LocalSlabGroup([DeviceSlab.create(gi, gd, T_l, R_l, cfg.ngf, cfg.alpha, lo, hi)
                                  for lo, hi in slabs])
        y = dev.to_device(identity_field_array(gd, dtype)) if y is None else _prolong_dev(y, prev, gd)
        setup_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        x, trace = lbfgs_minimize(obj, y.reshape(-1), cfg.lbfgs, cfg.stopping)
        y = x.reshape((3,) + gd.shape)
        prev = gd
        final_g = trace.records[-1].grad_inf if trace.records else 0.0
        report.levels.append(LevelReport(
            level_index=lvl, image_dims=gi.dims, def_dims=gd.dims, iterations=trace.iterations,
            stop_reason=trace.stop_reason, line_search_failed=trace.line_search_failed,
            records=trace.records, J_trace=list(trace.J_rows), final_grad_inf=final_g,
            seconds_setup=setup_s, seconds_optimize=time.perf_counter() - t0,
            evaluations=trace.evaluations))
        report.final_grad_inf = final_g
    report.seconds_total = time.perf_counter() - t_start
    return DeformationField(prev, dev.to_host(y) if np_out else y), report

"""Config-5 z-slab decomposition, host side, on CPU with the gloo backend (world size 2).

Each rank evaluates the NGF partial of its image z-slab (here with the CPU oracle
standing in for the sm_100a slab kernel), `SlabObjective` all-reduces grad D and D
and adds the curvature term; the result must equal the undivided objective on
every rank.  The GPU slab kernel itself is checked against the undivided fused
evaluation in tests/test_gpu_slab.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ngf_oracle as O
from paper_1812_06765_b200.distributed import SlabObjective, slab_ranges, weak_scaling_pairs


def _problem():
    gi = O.grid((20, 18, 16), (1.0, 1.1, 0.9), (0.0, -2.0, 1.0))
    gd = O.def_grid_for(gi, 4)
    R = O.smooth_random_volume(gi, 3)
    T = O.smooth_random_volume(gi, 4)
    y = O.smooth_random_field(gd, 5, 1.5)
    return gi, gd, R, T, y


class OracleSlab:
    """CPU oracle slab partial: distance terms and q restricted to image planes
    [zlo, zhi), pushed through G^T, J^T and P^T (ngf.py:83-134)."""

    def __init__(self, gi, gd, R, T, zlo, zhi, tau=10.0, rho=10.0, alpha=1.0):
        self.gi, self.gd, self.T, self.zlo, self.zhi = gi, gd, T, zlo, zhi
        self.image_grid, self.def_grid = gi, gd
        self.tau, self.rho, self.alpha = tau, rho, alpha
        self.gR, self.nR = O.ref_terms(R, gi, rho)

    def partial(self, x, grad, scal):
        y = x.numpy().reshape((3,) + O.shape_of(self.gd))
        yhat = O.apply_P(y, self.gd, self.gi)
        W, _ = O.warp(self.T, self.gi, yhat)
        gW = O.gradient(W, self.gi.spacing)
        r, nT = O._ratio(gW, self.gR, self.nR, self.tau, self.rho)
        sl = slice(self.zlo, self.zhi)
        D = O.cell_volume(self.gi) / 2 * float(np.sum(1 - r[sl] * r[sl]))
        coef = -O.cell_volume(self.gi) * r
        q = coef * (self.gR / (nT * self.nR) - r * gW / (nT * nT))
        mask = np.zeros(r.shape)
        mask[sl] = 1.0
        s = O.gradient_t(q * mask, self.gi.spacing)
        ghat = O.warp_jt(self.T, self.gi, yhat, s)
        grad.copy_(torch.from_numpy(O.apply_Pt(ghat, self.gd, self.gi).ravel()))
        scal[1] = D

    def finish(self, x, grad, scal):
        y = x.numpy().reshape((3,) + O.shape_of(self.gd))
        S = O.curvature_value(y, self.gd)
        grad += self.alpha * torch.from_numpy(O.curvature_gradient(y, self.gd).ravel())
        scal[0] = float(scal[1]) + self.alpha * S
        scal[2] = S


def _worker(rank, world, port, out, exchange="planes"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gi, gd, R, T, y = _problem()
        zlo, zhi = slab_ranges(gi.dims[2], gd.dims[2], world)[rank]
        obj = SlabObjective(OracleSlab(gi, gd, R, T, zlo, zhi), exchange=exchange)
        x = torch.from_numpy(y.ravel().copy())
        g = torch.zeros_like(x)
        sc = torch.zeros(3, dtype=torch.float64)
        obj.eval_device(x, g, sc)
        out[rank] = (sc.numpy().copy(), g.numpy().copy(), (zlo, zhi))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, exchange):
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_worker, args=(world, _free_port(), out, exchange), nprocs=world, join=True,
                           start_method="spawn")
        return dict(out)


@pytest.mark.parametrize("world,exchange", [(2, "planes"), (2, "allreduce"), (3, "planes")])
def test_slab_decomposition_gloo(world, exchange):
    res = _run(world, exchange)
    gi, gd, R, T, y = _problem()
    J, g = O.Objective(T, R, gd, gi)(y.ravel())
    slabs = [res[r][2] for r in range(world)]
    assert slabs[0][0] == 0 and slabs[-1][1] == gi.dims[2]
    assert all(slabs[r][1] == slabs[r + 1][0] for r in range(world - 1))
    for r in range(world):
        sc, gr, _ = res[r]
        assert abs(sc[0] - J) <= 1e-12 * abs(J)
        assert np.max(np.abs(gr - g)) <= 1e-11 * np.abs(g).max()
    # every rank holds the same result (replicated L-BFGS stays in lock-step)
    for r in range(1, world):
        assert np.array_equal(res[0][1], res[r][1]) and np.array_equal(res[0][0], res[r][0])


def test_slab_plane_layout_partitions_and_covers():
    from paper_1812_06765_b200.distributed import slab_plane_layout

    gi = O.grid((64, 64, 512), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = O.def_grid_for(gi, 4)
    slabs = slab_ranges(512, gd.dims[2], 8)
    windows, owned = slab_plane_layout(gi, gd, slabs)
    assert owned[0][0] == 0 and owned[-1][1] == gd.dims[2]
    assert all(owned[r][1] == owned[r + 1][0] for r in range(7))
    for (lo, hi), (wlo, whi) in zip(owned, windows):
        assert wlo <= lo and hi - 1 <= whi          # a rank's window covers its owned planes
        assert whi - wlo + 1 <= (hi - lo) + 4       # plus at most a couple of halo planes


def test_slab_ranges_align_to_deformation_cells():
    assert slab_ranges(512, 128, 8) == [(64 * r, 64 * (r + 1)) for r in range(8)]
    assert slab_ranges(256, 64, 3) == [(0, 84), (84, 172), (172, 256)]
    for lo, hi in slab_ranges(256, 64, 3)[:-1]:
        assert hi % 4 == 0
    assert slab_ranges(17, 5, 2)[-1][1] == 17
    with pytest.raises(ValueError):
        slab_ranges(4, 4, 8)


def test_weak_scaling_pair_assignment():
    assign = [weak_scaling_pairs(64, 8, r) for r in range(8)]
    assert sorted(p for a in assign for p in a) == list(range(64))
    assert all(len(a) == 8 for a in assign)
    assign = [weak_scaling_pairs(10, 4, r) for r in range(4)]
    assert sorted(p for a in assign for p in a) == list(range(10))


# ---------------------------------------------------------------------------------------
# Config 5 as a registration: one L-BFGS level driven over the slab objective (VERDICT r1
# item 4).  Every rank runs the reference's L-BFGS (oracle restatement of lbfgs.py:94-181)
# on the combined (J, grad J); the ranks stay in lock-step and their trace equals, bit for
# bit, the single-process evaluation of the same slabs (LocalSlabGroup), which in turn
# matches the undivided objective to rounding.

LBFGS_ITERS = 8


def _lbfgs_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gi, gd, R, T, y = _problem()
        zlo, zhi = slab_ranges(gi.dims[2], gd.dims[2], world)[rank]
        obj = SlabObjective(OracleSlab(gi, gd, R, T, zlo, zhi))
        x, recs, reason, failed = O.lbfgs(obj, y.ravel(), {"max_iterations": LBFGS_ITERS})
        out[rank] = (x, recs, reason, obj.evals)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_lbfgs_level_trace_identical(world):
    from paper_1812_06765_b200.distributed import LocalSlabGroup

    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_lbfgs_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                           start_method="spawn")
        res = dict(out)
    gi, gd, R, T, y = _problem()
    slabs = slab_ranges(gi.dims[2], gd.dims[2], world)
    local = LocalSlabGroup([OracleSlab(gi, gd, R, T, lo, hi) for lo, hi in slabs])
    x_l, recs_l, reason_l, _ = O.lbfgs(local, y.ravel(), {"max_iterations": LBFGS_ITERS})
    for r in range(world):
        x, recs, reason, evals = res[r]
        assert recs == recs_l and reason == reason_l, f"rank {r} trace differs"
        assert np.array_equal(x, x_l)
        assert evals == local.evals
    # the undivided objective: the same minimisation to rounding
    x_u, recs_u, _, _ = O.lbfgs(O.Objective(T, R, gd, gi), y.ravel(), {"max_iterations": LBFGS_ITERS})
    assert len(recs_u) == len(recs_l)
    for (_, Ja, *_), (_, Jb, *_) in zip(recs_u, recs_l):
        assert abs(Ja - Jb) <= 1e-9 * abs(Ja)
    assert np.max(np.abs(x_u - x_l)) <= 1e-7 * np.max(np.abs(x_u))


def test_combine_slab_partials_matches_sum():
    from paper_1812_06765_b200.distributed import combine_slab_partials, slab_plane_layout

    gi, gd, R, T, y = _problem()
    slabs = slab_ranges(gi.dims[2], gd.dims[2], 3)
    windows, owned = slab_plane_layout(gi, gd, slabs)
    nd = gd.dims
    rng = np.random.default_rng(0)
    parts = []
    for lo, hi in windows:
        p = np.zeros((3, nd[2], nd[1] * nd[0]))
        p[:, lo:hi + 1] = rng.standard_normal((3, hi + 1 - lo, nd[1] * nd[0]))
        parts.append(torch.from_numpy(p))
    got = combine_slab_partials(parts, windows, owned).numpy()
    want = sum(p.numpy() for p in parts)
    assert np.allclose(got, want, rtol=0, atol=1e-12)

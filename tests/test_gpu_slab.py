"""Config-5 z-slab mode of the fused kernel on one GPU: the sum of the slab partials
plus the curvature term equals the undivided fused evaluation and the oracle."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1812_06765_b200 as ngf  # noqa: E402
from oracle import ngf_oracle as O  # noqa: E402
from paper_1812_06765_b200.distributed import (DeviceSlab, SlabObjective, slab_plane_layout,  # noqa: E402
                                                slab_ranges)


@pytest.mark.parametrize("dims,ratio,world", [((64, 48, 40), 4, 2), ((48, 40, 37), 4, 3),
                                              ((40, 40, 40), 1, 4)])
def test_slab_partials_sum_to_full(dims, ratio, world):
    gi = ngf.Grid3(dims, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.deformation_grid_for(gi, ratio)
    R = ngf.smooth_random_volume(gi, seed=1).values.astype(np.float32)
    T = ngf.smooth_random_volume(gi, seed=2).values.astype(np.float32)
    y = ngf.smooth_random_field(gd, seed=3, amplitude_mm=2.0).field.astype(np.float32)
    plan = ngf.build_gather_plan(gd, gi)
    Td, Rd = torch.from_numpy(T).cuda(), torch.from_numpy(R).cuda()
    x = torch.from_numpy(y.ravel().copy()).cuda()

    full = ngf.LevelObjective.from_device(Td, Rd, plan, ngf.NgfParams(), 1.0)
    gf = torch.empty_like(x)
    sf = full.eval_device(x, gf).cpu().numpy().copy()

    gsum = torch.zeros_like(x)
    dsum = 0.0
    last = None
    slabs = slab_ranges(gi.dims[2], gd.dims[2], world)
    windows, _ = slab_plane_layout(gi, gd, slabs)
    for (zlo, zhi), (wlo, whi) in zip(slabs, windows):
        obj = ngf.LevelObjective.from_device(Td, Rd, plan, ngf.NgfParams(), 1.0)
        slab = DeviceSlab(obj.level, zlo, zhi)
        g = torch.empty_like(x)
        sc = torch.zeros(3, dtype=torch.float64, device="cuda")
        slab.partial(x, g, sc)
        # the plane exchange (SlabObjective) relies on the partial living in its window
        gp = g.view(3, gd.dims[2], -1)
        assert not torch.any(gp[:, :wlo]) and not torch.any(gp[:, whi + 1:]), (zlo, zhi, wlo, whi)
        gsum += g
        dsum += float(sc[1].item())
        last = slab
    sc = torch.tensor([0.0, dsum, 0.0], dtype=torch.float64, device="cuda")
    last.finish(x, gsum, sc)
    s = sc.cpu().numpy()
    assert abs(s[0] - sf[0]) <= 1e-5 * abs(sf[0])
    rel = (torch.linalg.norm(gsum - gf) / torch.linalg.norm(gf)).item()
    assert rel <= 1e-5
    J_ref, g_ref = O.Objective(T, R, O.grid(gd.dims, gd.spacing, gd.origin), O.grid(gi.dims))(y.ravel())
    assert abs(s[0] - J_ref) <= 1e-4 * abs(J_ref)
    g = gsum.cpu().numpy()
    assert np.linalg.norm(g - g_ref) / np.linalg.norm(g_ref) <= 1e-3


def test_slab_objective_without_process_group_equals_full():
    gi = ngf.Grid3((32, 32, 32), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    gd = ngf.deformation_grid_for(gi, 4)
    R = ngf.smooth_random_volume(gi, seed=4).values.astype(np.float32)
    T = ngf.smooth_random_volume(gi, seed=5).values.astype(np.float32)
    y = ngf.smooth_random_field(gd, seed=6, amplitude_mm=1.0).field.astype(np.float32)
    plan = ngf.build_gather_plan(gd, gi)
    Td, Rd = torch.from_numpy(T).cuda(), torch.from_numpy(R).cuda()
    x = torch.from_numpy(y.ravel().copy()).cuda()
    full = ngf.LevelObjective.from_device(Td, Rd, plan, ngf.NgfParams(), 1.0)
    gf = torch.empty_like(x)
    sf = full.eval_device(x, gf).cpu().numpy().copy()
    one = ngf.LevelObjective.from_device(Td, Rd, plan, ngf.NgfParams(), 1.0)
    obj = SlabObjective(DeviceSlab(one.level, 0, 32))  # one slab = whole volume
    g = torch.empty_like(x)
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    obj.eval_device(x, g, sc)
    assert torch.equal(g, gf)
    assert sc.cpu().numpy()[0] == sf[0]

"""Synthetic registration inputs (host numpy; test and benchmark data, not the hot path).

Two families:

* the reference's analytic sinusoid pattern and Gaussian-bump mapping
  (synthetic.py:25-110 of ngfreg), restated so identical inputs can be built on
  the GPU box, where the reference is not installed;
* `ct_pair`: the "thorax-like" / "CT-shaped" pairs of BASELINE.json configs 2-5
  (SURVEY.md §8(d)), which the reference does not ship.  The phantom is an
  analytic function of world position (body ellipsoid, two lungs, spine, a rib
  pattern, soft-tissue texture), so the template is sampled exactly at the
  mapped positions: R(x) = T(m(x)) with m the identity plus three smooth bumps.
"""

from __future__ import annotations

import numpy as np

from .geometry import DeformationField, Grid3, Image3, identity_field_array

__all__ = ["analytic_intensity", "gaussian_bump_mapping", "make_volume", "make_registration_pair",
           "probe_lattice", "smooth_random_volume", "smooth_random_field", "ct_phantom",
           "multi_bump_mapping", "ct_pair"]


def _coords(grid: Grid3):
    xs, ys, zs = (grid.axis_centers(a) for a in range(3))
    return xs[None, None, :], ys[None, :, None], zs[:, None, None]


def analytic_intensity(x, y, z, amplitude: float = 400.0, period_mm: float = 24.0):
    """Smooth pattern with gradients everywhere (reference synthetic.py:25-32)."""
    w = 2 * np.pi / period_mm
    a = np.sin(w * x) * np.cos(0.83 * w * y)
    b = np.sin(0.67 * w * y) * np.cos(1.19 * w * z)
    c = np.sin(0.91 * w * z) * np.cos(0.74 * w * x)
    return amplitude * (a + b + c) / 3.0


def make_volume(grid: Grid3, amplitude: float = 400.0, period_mm: float = 24.0) -> Image3:
    x, y, z = _coords(grid)
    return Image3(grid, analytic_intensity(x, y, z, amplitude, period_mm) + np.zeros(grid.shape))


def gaussian_bump_mapping(center, sigma_mm: float, amplitude_mm):
    """x -> x + a * exp(-|x-c|^2 / (2 sigma^2)) (reference synthetic.py:48-58)."""
    c = tuple(float(v) for v in center)
    a = tuple(float(v) for v in amplitude_mm)

    def mapping(x, y, z):
        e = np.exp(-((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2) / (2 * sigma_mm ** 2))
        return x + a[0] * e, y + a[1] * e, z + a[2] * e

    return mapping


def make_registration_pair(grid: Grid3, mapping, amplitude: float = 400.0, period_mm: float = 24.0):
    """T = pattern, R(x) = T(mapping(x)) (reference synthetic.py:61-69)."""
    x, y, z = _coords(grid)
    T = analytic_intensity(x, y, z, amplitude, period_mm) + np.zeros(grid.shape)
    R = analytic_intensity(*mapping(x, y, z), amplitude, period_mm) + np.zeros(grid.shape)
    return Image3(grid, R), Image3(grid, T)


def probe_lattice(grid: Grid3, n_per_axis: int = 5, margin: float = 0.25) -> np.ndarray:
    """(n^3, 3) lattice over the central part of the domain (reference synthetic.py:72-80)."""
    axes = [np.linspace(grid.origin[a] + margin * grid.extent[a],
                        grid.origin[a] + (1 - margin) * grid.extent[a], n_per_axis) for a in range(3)]
    gx, gy, gz = np.meshgrid(*axes, indexing="ij")
    return np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])


def smooth_random_volume(grid: Grid3, seed: int = 0, amplitude: float = 400.0,
                         smooth_passes: int = 3) -> Image3:
    """Gaussian noise box-filtered along each axis, scaled to `amplitude`
    (reference synthetic.py:83-100; same generator stream and filter order)."""
    v = np.random.default_rng(seed).standard_normal(grid.shape)
    for _ in range(smooth_passes):
        for ax in range(3):
            n = v.shape[ax]
            if n <= 2:
                continue
            prev = np.take(v, np.arange(0, n - 2), axis=ax)
            mid = np.take(v, np.arange(1, n - 1), axis=ax)
            nxt = np.take(v, np.arange(2, n), axis=ax)
            idx = [slice(None)] * 3
            idx[ax] = slice(1, n - 1)
            v[tuple(idx)] = (prev + mid + nxt) / 3
    v *= amplitude / max(np.abs(v).max(), 1e-12)
    return Image3(grid, v)


def smooth_random_field(grid: Grid3, seed: int = 0, amplitude_mm: float = 1.0) -> DeformationField:
    """Identity plus smooth random displacement (reference synthetic.py:103-110)."""
    rng = np.random.default_rng(seed)
    out = identity_field_array(grid)
    for c in range(3):
        out[c] += smooth_random_volume(grid, seed=int(rng.integers(1 << 31)),
                                       amplitude=amplitude_mm).values
    return DeformationField(grid, out)


# --------------------------------------------------------------------------- CT-like phantom

def _smoothstep(d, width):
    """0 outside (d > 0), 1 inside, smooth over `width` mm."""
    return 0.5 * (1.0 - np.tanh(d / width))


def ct_phantom(x, y, z, extent, edge_mm: float = 1.5):
    """Analytic thorax-like CT intensity (HU) at world positions; `extent` = (ex, ey, ez)."""
    ex, ey, ez = extent
    u = x / ex - 0.5
    v = y / ey - 0.5
    w = z / ez - 0.5
    scale = min(ex, ey)
    air = -1000.0
    # body: elliptic cylinder along z, rounded at the ends
    body_d = (np.sqrt((u / 0.42) ** 2 + (v / 0.32) ** 2) - 1.0) * 0.32 * scale
    body_d = np.maximum(body_d, (np.abs(w) - 0.47) * ez)
    body = _smoothstep(body_d, edge_mm)
    # lungs: two ellipsoids
    lung = np.zeros(np.broadcast_shapes(np.shape(u), np.shape(v), np.shape(w)))
    for sx in (-1.0, 1.0):
        d = (np.sqrt(((u - sx * 0.17) / 0.13) ** 2 + ((v + 0.02) / 0.2) ** 2 + (w / 0.33) ** 2)
             - 1.0) * 0.13 * scale
        lung = np.maximum(lung, _smoothstep(d, edge_mm))
    # spine: cylinder behind the lungs, vertebra pattern along z
    sp_d = (np.sqrt((u / 0.05) ** 2 + ((v - 0.21) / 0.05) ** 2) - 1.0) * 0.05 * scale
    spine = _smoothstep(sp_d, edge_mm) * (0.75 + 0.25 * np.cos(2 * np.pi * w * 12.0))
    # ribs: periodic shells around the body wall
    r = np.sqrt((u / 0.42) ** 2 + (v / 0.32) ** 2)
    shell = _smoothstep(np.abs(r - 0.9) * 0.32 * scale - 0.012 * scale, edge_mm)
    ribs = shell * np.clip(np.cos(2 * np.pi * w * 9.0), 0.0, None) ** 2
    # soft tissue texture so NGF sees gradients everywhere inside the body
    tex = 25.0 * np.sin(2 * np.pi * x / 19.0) * np.cos(2 * np.pi * y / 23.0) * np.sin(2 * np.pi * z / 29.0)
    hu = air + body * (1040.0 + tex)          # soft tissue ~ +40 HU
    hu = hu + body * lung * (-840.0 - tex)    # lungs ~ -800 HU
    hu = hu + body * np.maximum(spine, ribs) * 660.0  # bone ~ +700 HU
    return hu


def multi_bump_mapping(grid: Grid3, max_disp_vox: float = 6.0, seed: int = 0):
    """Identity plus three Gaussian bumps; largest |u| ~ max_disp_vox voxels."""
    rng = np.random.default_rng(seed)
    ext = np.array(grid.extent)
    lo = np.array(grid.origin) - np.array(grid.spacing) / 2
    h = float(min(grid.spacing))
    bumps = []
    for _ in range(3):
        c = lo + ext * rng.uniform(0.3, 0.7, 3)
        sigma = float(min(ext) * rng.uniform(0.12, 0.2))
        a = rng.standard_normal(3)
        a *= max_disp_vox * h / np.linalg.norm(a) * rng.uniform(0.6, 1.0)
        bumps.append((c, sigma, a))

    def mapping(x, y, z):
        ox, oy, oz = x + 0.0, y + 0.0, z + 0.0
        for c, s, a in bumps:
            e = np.exp(-((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2) / (2 * s * s))
            ox = ox + a[0] * e
            oy = oy + a[1] * e
            oz = oz + a[2] * e
        return ox, oy, oz

    return mapping


def ct_pair(n: int, spacing: float = 1.0, seed: int = 0, max_disp_vox: float = 6.0, dtype=np.float32):
    """Thorax-like pair on an n^3 grid: T = phantom, R(x) = T(m(x)).  Returns (R, T, mapping).

    Evaluated slab by slab in float64, stored as `dtype` (f32 halves host memory at 512^3)."""
    grid = Grid3((n, n, n), (spacing,) * 3, (0.0, 0.0, 0.0))
    mapping = multi_bump_mapping(grid, max_disp_vox, seed)
    ext = grid.extent
    xs, ys, zs = (grid.axis_centers(a) for a in range(3))
    R = np.empty(grid.shape, dtype)
    T = np.empty(grid.shape, dtype)
    X = xs[None, None, :]
    Y = ys[None, :, None]
    step = max(1, (1 << 22) // (n * n))
    for z0 in range(0, n, step):
        Z = zs[z0:z0 + step, None, None]
        T[z0:z0 + step] = ct_phantom(X, Y, Z, ext)
        mx, my, mz = mapping(X, Y, Z)
        R[z0:z0 + step] = ct_phantom(mx, my, mz, ext)
    return Image3(grid, R), Image3(grid, T), mapping

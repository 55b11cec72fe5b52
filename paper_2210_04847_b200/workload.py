"""Synthetic benchmark workloads — host-side harness, not the hot path.

The scene, camera and grid warm-up follow the reference CLI's ``bench`` command:

* scene: ``SolidSphere{c=(0.5,0.5,0.5), r=0.2, sigma=200, rgb=(0.8,0.25,0.25)}`` in the
  unit-cube ``AabbNormalize`` domain (CLI defaults, tools/voxmarch.cpp:41-47,54);
* rays: ``orbit_camera(unit box, angle 0, elevation 0.4, W=H, focal 1.1 W)``
  (tools/voxmarch.cpp:278-286) through ``look_at`` + ``generate_rays``
  (proj/src/scene_camera.cpp:24-63), near 0.2, far 1.0;
* grid: R^3, threshold 1e-2, 16 jittered updates with decay 0.95 and seeds drawn
  from ``Rng(5)`` (tools/voxmarch.cpp:269-276).

Ray generation restates the reference's double-precision arithmetic operation by
operation with numpy elementwise ops (no BLAS, so no FMA); tests/test_workload.py
checks it bit-for-bit against the reference's own ``generate_rays``.
"""
from __future__ import annotations

import math

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1

# BASELINE.json configs -> (rays per side, R, step, label)
CONFIGS = {
    1: dict(width=64, resolution=128, step=5e-3, label="bounded sphere, 4096 rays, 128^3"),
    2: dict(width=512, resolution=128, step=1.6914558667664816e-3,
            label="NeRF-Synthetic-shaped, 2^18 rays, 128^3, step sqrt(3)/1024"),
    4: dict(width=1024, resolution=128, step=5e-3, label="training loop, 2^20 rays/step, 128^3"),
    5: dict(width=2048, resolution=128, step=5e-3, label="large batch, 2^22 rays, 128^3"),
}

SPHERE = dict(center=(0.5, 0.5, 0.5), radius=0.2, sigma=200.0, rgb=(0.8, 0.25, 0.25))


def splitmix64(state: int):
    """rng.hpp:10-15 -> (new_state, output)."""
    state = (state + GOLDEN) & MASK
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return state, z ^ (z >> 31)


def mix_seed(a: int, b: int) -> int:
    """rng.hpp:17-20."""
    s = (a ^ ((b + GOLDEN + ((a << 6) & MASK) + (a >> 2)) & MASK)) & MASK
    return splitmix64(s)[1]


class Rng:
    """rng.hpp:25-48 (the constructor discards one draw)."""

    def __init__(self, seed: int = 0):
        self.state = seed & MASK
        self.state, _ = splitmix64(self.state)

    def next_u64(self) -> int:
        self.state, v = splitmix64(self.state)
        return v

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        u = float(self.next_u64() >> 11) * 2.0 ** -53
        return lo + (hi - lo) * u if (lo, hi) != (0.0, 1.0) else u


def grid_warmup_seeds(n_updates: int = 16, root: int = 5):
    """Seeds of build_grid's jittered updates: Rng(opt.seed=5).next_u64() each."""
    rng = Rng(root)
    return [rng.next_u64() for _ in range(n_updates)]


def _normalize(x, y, z):
    n = np.sqrt(x * x + y * y + z * z)
    return x / n, y / n, z / n


def orbit_rays(width: int, height: int | None = None, angle: float = 0.0,
               elevation: float = 0.4, near: float = 0.2, far: float = 1.0,
               box_min=(0.0, 0.0, 0.0), box_max=(1.0, 1.0, 1.0)):
    """Rays of the CLI bench camera, float64 AoS ``(origins[n,3], dirs[n,3])``."""
    height = width if height is None else height
    lo, hi = np.array(box_min, float), np.array(box_max, float)
    center = (lo + hi) * 0.5
    ext = hi - lo
    diag = math.sqrt(ext[0] * ext[0] + ext[1] * ext[1] + ext[2] * ext[2])
    radius = 0.6 * diag / math.sqrt(3.0)
    eye = center + np.array([radius * math.cos(angle) * math.cos(elevation),
                             radius * math.sin(angle) * math.cos(elevation),
                             radius * math.sin(elevation)])
    # look_at (scene_camera.cpp:24-44)
    off = eye - center
    n = math.sqrt(off[0] * off[0] + off[1] * off[1] + off[2] * off[2])
    zx, zy, zz = off[0] / n, off[1] / n, off[2] / n
    ux, uy, uz = 0.0, 0.0, 1.0
    xx, xy, xz = uy * zz - uz * zy, uz * zx - ux * zz, ux * zy - uy * zx
    n = math.sqrt(xx * xx + xy * xy + xz * xz)
    xx, xy, xz = xx / n, xy / n, xz / n
    yx, yy, yz = zy * xz - zz * xy, zz * xx - zx * xz, zx * xy - zy * xx
    focal = 1.1 * width
    # generate_rays (scene_camera.cpp:46-63): rotation rows are (x.x,y.x,z.x) ...
    cx, cy = 0.5 * width, 0.5 * height
    col = np.arange(width, dtype=np.float64)
    row = np.arange(height, dtype=np.float64)
    dcx = ((col + 0.5) - cx) / focal
    dcy = (cy - (row + 0.5)) / focal
    vx = np.broadcast_to(dcx[None, :], (height, width)).ravel()
    vy = np.broadcast_to(dcy[:, None], (height, width)).ravel()
    vz = -1.0
    wx = xx * vx + yx * vy + zx * vz
    wy = xy * vx + yy * vy + zy * vz
    wz = xz * vx + yz * vy + zz * vz
    dx, dy, dz = _normalize(wx, wy, wz)
    dirs = np.stack([dx, dy, dz], axis=1)
    origins = np.broadcast_to(eye, dirs.shape).copy()
    return origins, np.ascontiguousarray(dirs)


def upstream_grads(n_rays: int, seed: int = 113):
    """Upstream gradients d_color, d_opacity, d_depth ~ U(-1,1) (test_rendering.cpp:261-265
    pattern), drawn with numpy's PCG64 for speed at 2^22 rays."""
    g = np.random.default_rng(seed)
    return (g.uniform(-1, 1, (n_rays, 3)), g.uniform(-1, 1, n_rays), g.uniform(-1, 1, n_rays))

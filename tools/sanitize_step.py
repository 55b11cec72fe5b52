"""A small end-to-end run of every device entry point family, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per process): config-1-sized march +
shading + forward (fused, async), backward (short and long rays), the NerfAcc
operators, the cascade march and a grid update. Exits 0 when every result
matches its reference check."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_04847_b200 import api, workload  # noqa: E402
from paper_2210_04847_b200._lib import Contraction, Field, MarchConfig  # noqa: E402


def main():
    dev = api.Device(0)
    field = Field.sphere(**workload.SPHERE)
    grid = api.OccupancyGrid(64, Contraction.aabb(), dev=dev)
    for s in workload.grid_warmup_seeds(4, 5):
        grid.update_field(field, 0.95, s)
    o, d = workload.orbit_rays(64)
    rays = api.RayBatch.create(o, d, 0.2, 1.0, dev)
    p = api.march(rays, grid, field, MarchConfig(5e-3, 1e-4, 1e-2))
    rgb = np.random.default_rng(0).uniform(0, 1, (p.n_samples, 3))
    sig = np.random.default_rng(1).uniform(0, 50, p.n_samples)
    n = p.n_rays
    dc, do, dd = workload.upstream_grads(n, 3)
    api.render_forward(p, rgb, sig, dev=dev)
    api.render_backward(p, rgb, sig, dc, do, dd, dev=dev)
    api.render_backward(p, rgb, sig, dc, do, dd, dev=dev, dtype=np.float32)
    # long rays (k_backward_long) and a non-contiguous pack
    rng = np.random.default_rng(2)
    cnt = rng.integers(100, 400, 40).astype(np.uint32)
    off = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.uint32)
    s = int(cnt.sum())
    ts = np.sort(rng.uniform(0, 1, s))
    te = ts + 1e-3
    lp = api.PackedSamples(off, cnt, ts, te, np.zeros(s, np.uint32))
    lr, ls = rng.uniform(0, 1, (s, 3)), rng.uniform(0, 5, s)
    g = [rng.uniform(-1, 1, (40, 3)), rng.uniform(-1, 1, 40), rng.uniform(-1, 1, 40)]
    api.render_backward(lp, lr, ls, *g, dev=dev)
    rev = api.PackedSamples(off[::-1].copy(), cnt, ts, te, np.zeros(s, np.uint32))
    api.render_backward(rev, lr, ls, *g, dev=dev)
    w, t, a = api.render_weight_from_density(p, sig, dev=dev)
    api.render_weight_from_density_backward(p, sig, w, t, a, dev=dev)
    api.render_transmittance_from_alpha_backward(lp, rng.uniform(0, 0.2, s), rng.uniform(-1, 1, s), dev=dev)
    api.accumulate_along_rays(p, w, rgb, 3, dev=dev)
    api.ray_aabb_intersect(o, d, [[0, 0, 0, 1, 1, 1]], dev=dev)
    cas = api.Cascade(32, Contraction.aabb(), 3, dev=dev)
    cas.update_field(field, 0.95, 7)
    from paper_2210_04847_b200._lib import Rays, VMB_F64  # noqa: F401
    do_, dd_ = dev.upload(o), dev.upload(d)
    r = api.device_rays(dev, do_, dd_, 0.01, 100.0)
    api.march_cascade_device(dev, cas, r, field, MarchConfig(5e-3, 1e-4, 1e-2), api.DevicePacked.allocate(dev, n, 64 * n),
                             1 / 256)
    dev.sync()
    print("sanitize step ok", p.n_samples)


if __name__ == "__main__":
    main()

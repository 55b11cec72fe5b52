"""The benchmarked step alone, for ncu launch lists / captures: grid warm-up, then
`warmup` + 1 steps of (vmb_march_render_field -> vmb_render_backward) on one
stream (the same calls as bench.py's single-call step), then exit. The last
step's launches are the last ones in the list.

usage: python tools/profile_step.py [width=2048] [step=5e-3] [fusion=two|train] [field=sphere|checker|voxel]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_04847_b200 import api, workload  # noqa: E402
from paper_2210_04847_b200._lib import VMB_F32, Contraction, MarchConfig, Rays  # noqa: E402

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    step_size = float(sys.argv[2]) if len(sys.argv) > 2 else 5e-3
    fusion = sys.argv[3] if len(sys.argv) > 3 else "two"
    kind = sys.argv[4] if len(sys.argv) > 4 else "sphere"
    dev = api.Device(0)
    field, keep, _ = bench.make_field(kind, api, dev)
    cfg = MarchConfig(step_size, 1e-4, 1e-2)
    g = api.OccupancyGrid(128, Contraction.aabb(), dev=dev)
    for s in workload.grid_warmup_seeds(16, 5):
        g.update_field(field, 0.95, s)
    o, d = workload.orbit_rays(W)
    N = len(o)
    do_, dd_ = dev.upload(o.astype(np.float32)), dev.upload(d.astype(np.float32))
    rays = Rays(do_.ptr, dd_.ptr, VMB_F32, 0, N, 0.2, 1.0)
    p = api.march_device(dev, g, rays, field, cfg, api.DevicePacked.allocate(dev, N, 8 * N))
    cap = p.capacity
    rgb, sig = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)
    outs = [dev.empty(3 * N, np.float32), dev.empty(N, np.float32), dev.empty(N, np.float32)]
    ups = [dev.upload(x.astype(np.float32)) for x in workload.upstream_grads(N, 113)]
    gr, gs = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)
    n_dev = dev.zeros(1, np.uint64)
    for _ in range(4):
        if fusion == "train":
            api.march_render_backward_device(dev, g, rays, field, cfg, p, rgb, sig, *outs, *ups, gr, gs, n_dev)
        else:
            api.march_render_device(dev, g, rays, field, cfg, p, rgb, sig, *outs)
            api.render_backward_device(dev, p, rgb, sig, *ups, gr, gs)
    dev.sync()
    del keep


if __name__ == "__main__":
    main()

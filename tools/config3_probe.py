"""Config 3 stand-in timing: 2^20 rays from inside the unit ball, sphere
contraction, geometric step growth 1.01, near 0.01, far 100, 128^3 grid; march
(two-pass path: growth walks are sequential) + render forward + backward.
Exploration helper; prints one JSON line."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_04847_b200 import api, workload  # noqa: E402
from paper_2210_04847_b200._lib import VMB_F32, Contraction, Field, MarchConfig, Rays  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dev = api.Device(0)
con = Contraction.sphere((0.5, 0.5, 0.5), 0.5)
field = Field.sphere(radius=0.3, sigma=40.0)
g = api.OccupancyGrid(128, con, dev=dev)
for s in workload.grid_warmup_seeds(16, 5):
    g.update_field(field, 0.95, s)
o, d = workload.orbit_rays(W, near=0.01, far=100.0)
o[:] = [0.5, 0.5, 0.55]
N = len(o)
do_, dd_ = dev.upload(o.astype(np.float32)), dev.upload(d.astype(np.float32))
rays = Rays(do_.ptr, dd_.ptr, VMB_F32, 0, N, 0.01, 100.0)
cfg = MarchConfig(1.6914558667664816e-3, 1e-4, 1e-2, 2048, 1.01)
p = api.march_device(dev, g, rays, field, cfg, api.DevicePacked.allocate(dev, N, 64 * N))
cap = p.capacity
rgb, sig = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)
outs = [dev.empty(3 * N, np.float32), dev.empty(N, np.float32), dev.empty(N, np.float32)]
rng = np.random.default_rng(1)
ups = [dev.upload(rng.uniform(-1, 1, N * w).astype(np.float32)) for w in (3, 1, 1)]
gr, gs = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)


def step():
    api.march_render_device(dev, g, rays, field, cfg, p, rgb, sig, *outs)
    api.render_backward_device(dev, p, rgb, sig, *ups, gr, gs)


for _ in range(3):
    step()
dev.sync()
K = 10
dev.record(0)
for _ in range(K):
    step()
dev.record(1)
dev.sync()
ms = dev.elapsed_ms(0, 1) / K
print(json.dumps({"workload": f"config 3 stand-in: {N} rays, sphere contraction, growth 1.01, 128^3",
                  "ms_per_step": ms, "rays_per_s": N / (ms * 1e-3), "samples": p.n_samples,
                  "samples_per_s": p.n_samples / (ms * 1e-3)}))

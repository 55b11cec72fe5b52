import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2210_04847_b200 import api, workload
from paper_2210_04847_b200._lib import Contraction, Field, MarchConfig, VMB_F32, Rays, check
W = int(sys.argv[1])
dev = api.Device(0)
field = Field.sphere(**workload.SPHERE)
g = api.OccupancyGrid(128, Contraction.aabb(), dev=dev)
for s in workload.grid_warmup_seeds(16, 5):
    g.update_field(field, 0.95, s)
o, d = workload.orbit_rays(W)
N = len(o)
do_, dd_ = dev.upload(o.astype(np.float32)), dev.upload(d.astype(np.float32))
rays = Rays(do_.ptr, dd_.ptr, VMB_F32, 0, N, 0.2, 1.0)
cfg = MarchConfig(1.6914558667664816e-3, 1e-4, 1e-2)
p = api.march_device(dev, g, rays, field, cfg, api.DevicePacked.allocate(dev, N, 8 * N))
print("samples", p.n_samples, "max count", p.to_host().counts.max(), flush=True)
cap = p.capacity
rgb, sig = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)
outs = [dev.empty(3 * N, np.float32), dev.empty(N, np.float32), dev.empty(N, np.float32)]
api.march_render_device(dev, g, rays, field, cfg, p, rgb, sig, *outs)
dev.sync()
print("ok render", flush=True)

"""A/B of the config 5 resident step: two calls per sub-batch (march_render ->
render_backward) vs the fused training step, for several stream/sub-batch
schedules. Exploration helper; prints one JSON line per schedule."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_04847_b200 import api, workload  # noqa: E402
from paper_2210_04847_b200._lib import Contraction, Field, MarchConfig  # noqa: E402
from paper_2210_04847_b200.pipeline import ResidentPipeline  # noqa: E402

dev = api.Device(0)
field = Field.sphere(**workload.SPHERE)
cfg = MarchConfig(5e-3, 1e-4, 1e-2)
g = api.OccupancyGrid(128, Contraction.aabb(), dev=dev)
for s in workload.grid_warmup_seeds(16, 5):
    g.update_field(field, 0.95, s)
W = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
o, d = workload.orbit_rays(W)
N = len(o)
rays = (dev.upload(o.astype(np.float32)), dev.upload(d.astype(np.float32)))
ups = [dev.upload(x.astype(np.float32)) for x in workload.upstream_grads(N, 113)]
res = {}
for train in (False, True):
    for S, K in ((1, 1), (2, 2), (3, 2), (2, 4), (4, 4)):
        pipe = ResidentPipeline(S, K, api, dev, g, field, cfg, rays, ups, N, 6 * N, train=train)
        pipe.run(3)
        pipe.sync()
        pipe.begin(0)
        pipe.run(20)
        pipe.end(1)
        pipe.sync()
        ms = dev.elapsed_ms(0, 1) / 20
        total = pipe.check()
        if K <= S:
            res[(train, S, K)] = [pipe.chunk_outputs(k) for k in range(K)]
        print(json.dumps({"train": train, "streams": S, "chunks": K, "ms_per_step": ms, "rays_per_s": N / ms * 1e3,
                          "samples": total}), flush=True)
a, b = res[(False, 2, 2)], res[(True, 2, 2)]
for x, y in zip(a, b):
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices", "rgb", "sig"):
        assert np.array_equal(x[k], y[k]), k
    for k in ("grgb", "gsig"):
        err = np.abs(x[k].astype(np.float64) - y[k].astype(np.float64))
        tol = 1e-5 * np.maximum(np.abs(x[k]), np.abs(y[k])) + 1e-8
        assert (err <= tol).all(), (k, err.max())
print("fused == two calls")

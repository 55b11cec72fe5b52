"""Experiment: the resident config-5 step as K sub-batches over S contexts (streams),
kernels of different sub-batches free to overlap. Prints ms/step per (S, K).
Exploration helper, not the benchmark."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_04847_b200 import api, workload  # noqa: E402
from paper_2210_04847_b200._lib import VMB_F32, Contraction, Field, MarchConfig, Rays, check  # noqa: E402

SCENE = dict(center=(0.5, 0.5, 0.5), radius=0.2, sigma=200.0, rgb=(0.8, 0.25, 0.25))
dev = api.Device(0)
L = dev.lib
field = Field.sphere(**SCENE)
cfg = MarchConfig(5e-3, 1e-4, 1e-2)
grid = api.OccupancyGrid(128, Contraction.aabb(), dev=dev)
for s in workload.grid_warmup_seeds(16, 5):
    grid.update_field(field, 0.95, s)
o64, d64 = workload.orbit_rays(2048)
N = len(o64)
o_, d_ = dev.upload(o64.astype(np.float32)), dev.upload(d64.astype(np.float32))
dc, do, dd = workload.upstream_grads(N, 113)
ups = [dev.upload(x.astype(np.float32)) for x in (dc, do, dd)]
widths = [3, 1, 1]
configs = [tuple(int(v) for v in a.split("x")) for a in (sys.argv[1:] or ["1x1", "2x2", "2x4", "2x8", "3x6", "4x8"])]
pool = []
for S, K in configs:
    while len(pool) < S:
        pool.append(api.Device(0) if pool else dev)
    bounds = [(N * i // K, N * (i + 1) // K) for i in range(K)]
    cmax = max(e - b for b, e in bounds)
    cap = 8 * cmax
    bufs = []
    for cx in pool[:S]:
        bufs.append(dict(packed=api.DevicePacked.allocate(cx, cmax, cap), n_dev=cx.zeros(K, np.uint64),
                         rgb=cx.empty(cap * 3, np.float32), sig=cx.empty(cap, np.float32),
                         grgb=cx.empty(cap * 3, np.float32), gsig=cx.empty(cap, np.float32),
                         outs=[cx.empty(cmax * w, np.float32) for w in widths]))

    def chunk(k):
        ci = k % S
        cx, bf = pool[ci], bufs[ci]
        b, e = bounds[k]
        rays = Rays(o_.ptr + 12 * b, d_.ptr + 12 * b, VMB_F32, 0, e - b, 0.2, 1.0)
        pk = bf["packed"]
        smp = pk.samples_struct()
        check(L.vmb_march_render_field_async(cx.h, grid.h, C.byref(rays), C.byref(field), C.byref(cfg),
                                             C.byref(smp), bf["rgb"].ptr, bf["sig"].ptr, bf["outs"][0].ptr,
                                             bf["outs"][1].ptr, bf["outs"][2].ptr, VMB_F32, 0.0,
                                             bf["n_dev"].ptr + 8 * k))
        pk.n_samples = pk.capacity
        ua = [u.ptr + 4 * w * b for u, w in zip(ups, widths)]
        uarr = [type("A", (), {"ptr": p})() for p in ua]
        api.render_backward_device(cx, pk, bf["rgb"], bf["sig"], *uarr, bf["grgb"], bf["gsig"])

    def run(steps):
        for _ in range(steps):
            for k in range(K):
                chunk(k)

    run(3)
    for cx in pool[:S]:
        cx.sync()
    steps = 20
    dev.record(7)
    for cx in pool[1:S]:
        check(L.vmb_ctx_wait(cx.h, dev.h, 9))
    run(steps)
    for i, cx in enumerate(pool[1:S]):
        check(L.vmb_ctx_wait(dev.h, cx.h, 9 + i))
    dev.record(8)
    for cx in pool[:S]:
        cx.sync()
    for cx, bf in zip(pool[:S], bufs):
        check(L.vmb_march_check(cx.h))
    print(f"S={S} K={K} env={ {k: v for k, v in os.environ.items() if k.startswith('VMB_')} } "
          f"ms/step={dev.elapsed_ms(7, 8) / steps:.4f}", flush=True)

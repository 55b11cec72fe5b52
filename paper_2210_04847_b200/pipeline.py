"""The resident training step of the benchmark as a reusable host schedule.

A batch of rays already in HBM is marched + shaded + composited
(vmb_march_render_field_async) and differentiated (vmb_render_backward) as K
contiguous ray sub-batches served round-robin by S contexts (streams); bench.py
times it and tests/test_gpu_fullsize.py checks its outputs against the
reference at the benchmarked sizes. Host plumbing over the C ABI only.
"""
import ctypes as C

import numpy as np


class ResidentPipeline:
    """The resident step (rays, upstream gradients, outputs in HBM) as `--chunks`
    contiguous ray sub-batches served round-robin by `--streams` contexts, each
    sub-batch one vmb_march_render_field_async + vmb_render_backward pair on its
    context's stream. Sub-batches of different streams overlap on the device (one
    sub-batch's expansion/backward fills the SMs the other's walk tail leaves idle).
    Per-ray outputs land in full-batch arrays, so they can be compared with the
    single-call step bit for bit."""

    def __init__(self, streams, chunks, api, dev, grid, field, cfg, rays_dev, ups_dev, N, total_samples,
                 train=False):
        from paper_2210_04847_b200._lib import VMB_F32
        self.api, self.dev, self.grid, self.field, self.cfg = api, dev, grid, field, cfg
        self.L = dev.lib
        self.S, self.K = max(1, streams), max(1, chunks)
        self.train = train  # one vmb_march_render_backward_field_async per sub-batch
        self.N = N
        self.bounds = [(N * i // self.K, N * (i + 1) // self.K) for i in range(self.K)]
        cmax = max(e - b for b, e in self.bounds)
        cap = total_samples + 1024  # no sub-batch holds more samples than the whole batch
        self.ctxs = [dev] + [api.Device(dev.index) for _ in range(self.S - 1)]
        self.rays_dev, self.ups_dev = rays_dev, ups_dev
        self.outs = [dev.empty(N * w, np.float32) for w in (3, 1, 1)]
        self.n_dev = dev.zeros(self.K, np.uint64)
        self.bufs = [dict(packed=api.DevicePacked.allocate(cx, cmax, cap),
                          rgb=cx.empty(cap * 3, np.float32), sig=cx.empty(cap, np.float32),
                          grgb=cx.empty(cap * 3, np.float32), gsig=cx.empty(cap, np.float32))
                     for cx in self.ctxs]
        self.cap = cap
        self.VMB_F32 = VMB_F32

    def chunk(self, k):
        from paper_2210_04847_b200._lib import Rays, check

        class Ptr:  # a device pointer with the DeviceArray interface the api needs
            def __init__(self, ptr):
                self.ptr = ptr

        ci = k % self.S
        cx, bf = self.ctxs[ci], self.bufs[ci]
        b, e = self.bounds[k]
        o, d = self.rays_dev
        rays = Rays(o.ptr + 12 * b, d.ptr + 12 * b, self.VMB_F32, 0, e - b, 0.2, 1.0)
        pk = bf["packed"]
        smp = pk.samples_struct()
        outs = [a.ptr + 4 * w * b for a, w in zip(self.outs, (3, 1, 1))]
        ups = [Ptr(u.ptr + 4 * w * b) for u, w in zip(self.ups_dev, (3, 1, 1))]
        if self.train:
            check(self.L.vmb_march_render_backward_field_async(
                cx.h, self.grid.h, C.byref(rays), C.byref(self.field), C.byref(self.cfg), C.byref(smp),
                bf["rgb"].ptr, bf["sig"].ptr, outs[0], outs[1], outs[2], ups[0].ptr, ups[1].ptr, ups[2].ptr,
                bf["grgb"].ptr, bf["gsig"].ptr, self.VMB_F32, 0.0, self.n_dev.ptr + 8 * k))
            pk.n_samples = pk.capacity
            return
        check(self.L.vmb_march_render_field_async(
            cx.h, self.grid.h, C.byref(rays), C.byref(self.field), C.byref(self.cfg), C.byref(smp),
            bf["rgb"].ptr, bf["sig"].ptr, outs[0], outs[1], outs[2], self.VMB_F32, 0.0, self.n_dev.ptr + 8 * k))
        pk.n_samples = pk.capacity
        self.api.render_backward_device(cx, pk, bf["rgb"], bf["sig"], *ups, bf["grgb"], bf["gsig"])

    def run(self, steps=1, pre_step=None):
        """`pre_step()` (e.g. config 4's grid update) runs on context 0 before each
        step's sub-batches, ordered after every stream's previous work and before
        their next (the grid is read by every stream's walk)."""
        from paper_2210_04847_b200._lib import check
        for _ in range(steps):
            if pre_step is not None and pre_step(dry=True):
                for i, cx in enumerate(self.ctxs[1:]):
                    check(self.L.vmb_ctx_wait(self.dev.h, cx.h, 21 + (i % 8)))
                pre_step()
                for cx in self.ctxs[1:]:
                    check(self.L.vmb_ctx_wait(cx.h, self.dev.h, 20))
            for k in range(self.K):
                self.chunk(k)

    def begin(self, slot):
        """event `slot` on context 0; every other stream waits for it"""
        from paper_2210_04847_b200._lib import check
        self.dev.record(slot)
        for cx in self.ctxs[1:]:
            check(self.L.vmb_ctx_wait(cx.h, self.dev.h, 12))

    def end(self, slot):
        """context 0 waits for every other stream, then records `slot`"""
        from paper_2210_04847_b200._lib import check
        for i, cx in enumerate(self.ctxs[1:]):
            check(self.L.vmb_ctx_wait(self.dev.h, cx.h, 13 + (i % 8)))
        self.dev.record(slot)

    def sync(self):
        for cx in self.ctxs:
            cx.sync()

    def check(self):
        """deferred march errors; every sub-batch fitted its sample buffers; total samples"""
        from paper_2210_04847_b200._lib import check
        for cx in self.ctxs:
            check(self.L.vmb_march_check(cx.h))
        n = self.n_dev.numpy()
        assert int(n.max()) <= self.cap, "a sub-batch exceeded its sample capacity"
        return int(n.sum())

    def chunk_outputs(self, k):
        """Host copies of sub-batch k's packed samples, shading and gradients
        (valid while K <= S: each context's buffers then hold one sub-batch)."""
        assert self.K <= self.S, "sub-batch buffers are reused when K > S"
        cx, bf = self.ctxs[k % self.S], self.bufs[k % self.S]
        n = int(self.n_dev.numpy()[k])
        pk = bf["packed"]
        b, e = self.bounds[k]
        m = e - b
        out = dict(offsets=pk.offsets.numpy(m), counts=pk.counts.numpy(m),
                   t_starts=pk.t_starts.numpy(n), t_ends=pk.t_ends.numpy(n),
                   ray_indices=pk.ray_indices.numpy(n),
                   rgb=bf["rgb"].numpy(3 * n).reshape(-1, 3), sig=bf["sig"].numpy(n),
                   grgb=bf["grgb"].numpy(3 * n).reshape(-1, 3), gsig=bf["gsig"].numpy(n))
        return out

    def outputs(self):
        """color [N,3], opacity [N], depth [N] of the whole batch (host)."""
        c, o, d = self.outs
        return c.numpy(3 * self.N).reshape(-1, 3), o.numpy(self.N), d.numpy(self.N)

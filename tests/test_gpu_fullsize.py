"""The benchmarked composition, at the benchmarked sizes, against the reference.

bench.py times config 5 as: 2^22 f32 orbit-camera rays in HBM ->
vmb_march_render_field_async (walk + scan + expansion + shading + forward) and
vmb_render_backward, as 2 contiguous sub-batches over 2 streams
(paper_2210_04847_b200/pipeline.py). These tests run exactly that schedule and
compare every output with the reference's own CPU code (oracle/_ref, all host
threads) on the same rays widened to f64 (exact), the same grid and the same
upstream gradients:

  * packing bit-exact: counts, offsets (sub-batch offsets + the previous
    sub-batches' totals), t_starts, t_ends, ray_indices (+ the sub-batch's first
    ray), and the sample total S;
  * shading bit-exact after the f32 rounding of the attribute dtype;
  * color/opacity/depth and d_rgb/d_sigma within rtol 1e-5 (atol 1e-8), the
    tolerance of rendering.cpp's own tests (close_rel, test_rendering.cpp:67-69).

Config 2 (2^18 rays, step sqrt(3)/1024) and the config 3 stand-in (2^20 rays,
sphere contraction, growth 1.01) run the same way through the single-call path.
"""
import os

import numpy as np
import pytest

from oracle import Oracle, available
from oracle import oracle as O
from paper_2210_04847_b200 import api, workload
from paper_2210_04847_b200._lib import VMB_F32, Contraction, Field, MarchConfig, Rays
from paper_2210_04847_b200.pipeline import ResidentPipeline

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not available("ref") and not available("port"),
                                                  reason="oracle not built")]
RTOL, ATOL = 1e-5, 1e-8
THREADS = os.cpu_count() or 1


def close(a, b, what):
    a, b = np.asarray(a, float), np.asarray(b, float)
    assert a.shape == b.shape, what
    tol = np.maximum(RTOL * np.maximum(np.abs(a), np.abs(b)), ATOL)
    bad = np.abs(a - b) > tol
    assert not bad.any(), f"{what}: {bad.sum()} mismatches, worst {np.abs(a - b).max()}"


@pytest.fixture(scope="module")
def dev():
    return api.Device(0)


@pytest.fixture(scope="module")
def orc():
    return Oracle("ref") if available("ref") else Oracle("port")


def ofield(f: Field):
    o = O.Field()
    for name, _ in Field._fields_:
        setattr(o, name, getattr(f, name))
    return o


def grids(dev, orc, res, con, ocon, field):
    g = api.OccupancyGrid(res, con, dev=dev)
    og = orc.grid(res, ocon)
    for s in workload.grid_warmup_seeds(16, 5):
        g.update_field(field, 0.95, s)
        og.update_field(ofield(field), 0.95, s)
    assert np.array_equal(g.bits(), og.bits())
    return g, og


def reference_step(orc, og, field, o64, d64, near, far, cfg, ups64):
    ref = orc.march_field(o64, d64, near, far, og, ofield(field),
                          O.MarchConfig(cfg.step_size, cfg.early_stop_eps, cfg.alpha_thre,
                                        cfg.max_samples_per_ray, cfg.unbounded_step_growth), THREADS)
    rgb, sig = orc.shade(o64, d64, ref, ofield(field))
    rgb32 = rgb.astype(np.float32).astype(np.float64)
    sig32 = sig.astype(np.float32).astype(np.float64)
    fwd = orc.render_forward(ref, rgb32, sig32, THREADS)
    bwd = orc.render_backward(ref, rgb32, sig32, *ups64, THREADS)
    return ref, rgb32, sig32, fwd, bwd


@pytest.mark.parametrize("res", [128, 256])
def test_config5_pipelined_step_matches_reference(dev, orc, res):
    field = Field.sphere(**workload.SPHERE)
    cfg = MarchConfig(5e-3, 1e-4, 1e-2)
    g, og = grids(dev, orc, res, Contraction.aabb(), O.Contraction.aabb(), field)
    o, d = workload.orbit_rays(2048)
    N = len(o)
    assert N == 1 << 22
    o32, d32 = o.astype(np.float32), d.astype(np.float32)
    dc, do, dd = workload.upstream_grads(N, 113)
    ups32 = [x.astype(np.float32) for x in (dc, do, dd)]
    rays_dev = (dev.upload(o32), dev.upload(d32))
    ups_dev = [dev.upload(x) for x in ups32]
    pipe = ResidentPipeline(2, 2, api, dev, g, field, cfg, rays_dev, ups_dev, N, 6 * N)
    pipe.run(1)
    pipe.sync()
    S = pipe.check()

    ups64 = [x.astype(np.float64) for x in ups32]
    ref, rgb32, sig32, fwd, bwd = reference_step(orc, og, field, o32.astype(np.float64),
                                                 d32.astype(np.float64), 0.2, 1.0, cfg, ups64)
    assert S == ref.n_samples
    if res == 128:
        # f32 rays of the bench (the f64 rays of SURVEY §8 give 19,805,539)
        assert S == 19_805_543
    base = 0
    for k, (b, e) in enumerate(pipe.bounds):
        c = pipe.chunk_outputs(k)
        n = len(c["t_starts"])
        assert np.array_equal(c["counts"], ref.counts[b:e])
        assert np.array_equal(c["offsets"].astype(np.int64) + base, ref.offsets[b:e].astype(np.int64))
        sl = slice(base, base + n)
        assert np.array_equal(c["t_starts"], ref.t_starts[sl])
        assert np.array_equal(c["t_ends"], ref.t_ends[sl])
        assert np.array_equal(c["ray_indices"].astype(np.int64) + b, ref.ray_indices[sl].astype(np.int64))
        assert np.array_equal(c["rgb"].astype(np.float64), rgb32[sl])
        assert np.array_equal(c["sig"].astype(np.float64), sig32[sl])
        close(c["grgb"], bwd[0][sl], "d_rgb")
        close(c["gsig"], bwd[1][sl], "d_sigma")
        base += n
    assert base == S
    for got, want, what in zip(pipe.outputs(), fwd, ("color", "opacity", "depth")):
        close(got, want, what)


def _single_call(dev, g, field, cfg, o32, d32, near, far, ups32):
    N = len(o32)
    do_, dd_ = dev.upload(o32), dev.upload(d32)
    rays = Rays(do_.ptr, dd_.ptr, VMB_F32, 0, N, near, far)
    p = api.march_device(dev, g, rays, field, cfg, api.DevicePacked.allocate(dev, N, 8 * N))
    cap = p.capacity
    rgb, sig = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)
    outs = [dev.empty(3 * N, np.float32), dev.empty(N, np.float32), dev.empty(N, np.float32)]
    api.march_render_device(dev, g, rays, field, cfg, p, rgb, sig, *outs)
    ups = [dev.upload(x) for x in ups32]
    gr, gs = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)
    api.render_backward_device(dev, p, rgb, sig, *ups, gr, gs)
    s = p.n_samples
    return (p.to_host(), rgb.numpy(3 * s).reshape(-1, 3), sig.numpy(s),
            [outs[0].numpy(3 * N).reshape(-1, 3), outs[1].numpy(N), outs[2].numpy(N)],
            gr.numpy(3 * s).reshape(-1, 3), gs.numpy(s))


def _compare(got, ref, rgb32, sig32, fwd, bwd):
    p, rgb, sig, outs, gr, gs = got
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(p, k), getattr(ref, k)), k
    assert np.array_equal(rgb.astype(np.float64), rgb32)
    assert np.array_equal(sig.astype(np.float64), sig32)
    for a, b, what in zip(outs, fwd, ("color", "opacity", "depth")):
        close(a, b, what)
    close(gr, bwd[0], "d_rgb")
    close(gs, bwd[1], "d_sigma")


def test_config2_full_size_matches_reference(dev, orc):
    """BASELINE config 2: 2^18 rays, 128^3, step sqrt(3)/1024 (28 kept samples on a
    sphere ray: every hitting ray fills most of the walk's 32-sample buffer)."""
    field = Field.sphere(**workload.SPHERE)
    cfg = MarchConfig(1.6914558667664816e-3, 1e-4, 1e-2)
    g, og = grids(dev, orc, 128, Contraction.aabb(), O.Contraction.aabb(), field)
    o, d = workload.orbit_rays(512)
    o32, d32 = o.astype(np.float32), d.astype(np.float32)
    ups32 = [x.astype(np.float32) for x in workload.upstream_grads(len(o), 7)]
    got = _single_call(dev, g, field, cfg, o32, d32, 0.2, 1.0, ups32)
    ref = reference_step(orc, og, field, o32.astype(np.float64), d32.astype(np.float64), 0.2, 1.0, cfg,
                         [x.astype(np.float64) for x in ups32])
    _compare(got, *ref)


def test_config3_standin_full_size_matches_reference(dev, orc):
    """Config 3 stand-in (tools/config3_probe.py, bench --config 3): 2^20 rays from
    inside the unit ball, sphere contraction r=0.5, growth 1.01, near 0.01, far 100,
    128^3 — the two-pass growth walk, the windowed shade+forward and the long-ray
    backward (every ray is longer than a tile)."""
    field = Field.sphere(radius=0.3, sigma=40.0)
    cfg = MarchConfig(1.6914558667664816e-3, 1e-4, 1e-2, 2048, 1.01)
    g, og = grids(dev, orc, 128, Contraction.sphere((0.5, 0.5, 0.5), 0.5),
                  O.Contraction.sphere((0.5, 0.5, 0.5), 0.5), field)
    o, d = workload.orbit_rays(1024, near=0.01, far=100.0)
    o[:] = [0.5, 0.5, 0.55]
    o32, d32 = o.astype(np.float32), d.astype(np.float32)
    ups32 = [x.astype(np.float32) for x in workload.upstream_grads(len(o), 9)]
    got = _single_call(dev, g, field, cfg, o32, d32, 0.01, 100.0, ups32)
    ref = reference_step(orc, og, field, o32.astype(np.float64), d32.astype(np.float64), 0.01, 100.0, cfg,
                         [x.astype(np.float64) for x in ups32])
    _compare(got, *ref)


def test_config3_cascade_full_size_matches_port(dev):
    """bench.py --workload config3 at full size (2^20 rays, 4 cascaded 128^3 levels,
    cone 1/256): the device's whole batch, checked on every 16th ray against the
    port's sequential cascade march (oracle/vm_oracle.c vmo_march_cascade; the
    reference has no cascade), bit-exact, plus shading and the
    forward/backward of those rays against the port's render functions."""
    import math
    from paper_2210_04847_b200._lib import MarchStats
    port = Oracle("port")
    field = Field.sphere(radius=0.3, sigma=40.0)
    cfg = MarchConfig(math.sqrt(3.0) / 1024, 1e-4, 1e-2, 4096, 1.0)
    cas = api.Cascade(128, Contraction.aabb((0, 0, 0), (1, 1, 1)), 4, dev=dev)
    pg = []
    for level in range(4):
        con = Contraction()
        import ctypes as C
        dev.lib.vmb_cascade_level_box(C.byref(Contraction.aabb((0, 0, 0), (1, 1, 1))), level, C.byref(con))
        pg.append(port.grid(128, O.Contraction.aabb(tuple(con.box_min), tuple(con.box_max))))
    for s in workload.grid_warmup_seeds(16, 5):
        cas.update_field(field, 0.95, s)
        for g in pg:
            g.update_field(ofield(field), 0.95, s)
    for g, q in zip(cas.grids, pg):
        assert np.array_equal(g.bits(), q.bits())
    o, d = workload.orbit_rays(1024, near=0.01, far=100.0)
    N = len(o)
    o32, d32 = o.astype(np.float32), d.astype(np.float32)
    do_, dd_ = dev.upload(o32), dev.upload(d32)
    rays = Rays(do_.ptr, dd_.ptr, VMB_F32, 0, N, 0.01, 100.0)
    st = MarchStats()
    p = api.march_cascade_device(dev, cas, rays, field, cfg, api.DevicePacked.allocate(dev, N, 64 * N), 1 / 256,
                                 1e10, st)
    cap = p.capacity
    rgb, sig = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)
    outs = [dev.empty(3 * N, np.float32), dev.empty(N, np.float32), dev.empty(N, np.float32)]
    api.march_render_cascade_device(dev, cas, rays, field, cfg, p, rgb, sig, *outs, cone_angle=1 / 256)
    ups32 = [x.astype(np.float32) for x in workload.upstream_grads(N, 31)]
    ups = [dev.upload(x) for x in ups32]
    gr, gs = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)
    api.render_backward_device(dev, p, rgb, sig, *ups, gr, gs)
    h = p.to_host()
    S = h.n_samples
    sel = np.arange(0, N, 16)
    ref = port.march_cascade(o32[sel].astype(np.float64), d32[sel].astype(np.float64), 0.01, 100.0, pg[0], pg[1:],
                             ofield(field), O.MarchConfig(cfg.step_size, 1e-4, 1e-2, 4096, 1.0), 1 / 256, 1e10)
    assert np.array_equal(h.counts[sel], ref.counts)
    idx = np.concatenate([np.arange(h.offsets[r], h.offsets[r] + h.counts[r]) for r in sel])
    assert np.array_equal(h.t_starts[idx], ref.t_starts) and np.array_equal(h.t_ends[idx], ref.t_ends)
    assert np.array_equal(h.ray_indices[idx], sel[ref.ray_indices])
    prgb, psig = port.shade(o32[sel].astype(np.float64), d32[sel].astype(np.float64), ref, ofield(field))
    r32 = prgb.astype(np.float32).astype(np.float64)
    s32 = psig.astype(np.float32).astype(np.float64)
    assert np.array_equal(rgb.numpy(3 * S).reshape(-1, 3)[idx].astype(np.float64), r32)
    assert np.array_equal(sig.numpy(S)[idx].astype(np.float64), s32)
    fwd = port.render_forward(ref, r32, s32)
    for a, b, what in zip(outs, fwd, ("color", "opacity", "depth")):
        got = a.numpy().reshape(N, -1)[sel].reshape(np.shape(b))
        close(got, b, what)
    bwd = port.render_backward(ref, r32, s32, *[u[sel].astype(np.float64) for u in ups32])
    close(gr.numpy(3 * S).reshape(-1, 3)[idx], bwd[0], "d_rgb")
    close(gs.numpy(S)[idx], bwd[1], "d_sigma")

"""vmb_march_field_shaded == vmb_march_field followed by vmb_shade_field, bit for bit
(same packed samples, same rgb/sigma), for f32/f64 attributes, the fused
single-pass marcher, its overflow fixup and the two-pass (growth) path."""
import numpy as np
import pytest

from paper_2210_04847_b200 import api, workload
from paper_2210_04847_b200._lib import VMB_F32, VMB_F64, Contraction, Field, MarchConfig, Rays

pytestmark = pytest.mark.gpu


def _rays(dev, o, d, near, far, dtype):
    do_, dd_ = dev.upload(o.astype(dtype)), dev.upload(d.astype(dtype))
    return Rays(do_.ptr, dd_.ptr, VMB_F32 if dtype == np.float32 else VMB_F64, 0, len(o), near, far), (do_, dd_)


def _both(dev, grid, rays, field, cfg, n, attr_dtype, time=0.0):
    a = api.march_device(dev, grid, rays, field, cfg, api.DevicePacked.allocate(dev, n, 8 * n + 1024))
    cap = a.capacity  # march_device grows the buffers to the exact need
    rgb_a, sig_a = dev.empty(cap * 3, attr_dtype), dev.empty(cap, attr_dtype)
    api.shade_device(dev, rays, field, a, rgb_a, sig_a, time)
    b = api.DevicePacked.allocate(dev, n, cap)
    rgb_b, sig_b = dev.empty(cap * 3, attr_dtype), dev.empty(cap, attr_dtype)
    api.march_shaded_device(dev, grid, rays, field, cfg, b, rgb_b, sig_b, time)
    ha, hb = a.to_host(), b.to_host()
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(ha, k), getattr(hb, k)), k
    s = a.n_samples
    assert s > 0
    assert np.array_equal(rgb_a.numpy(3 * s), rgb_b.numpy(3 * s))
    assert np.array_equal(sig_a.numpy(s), sig_b.numpy(s))


@pytest.mark.parametrize("ray_dtype,attr_dtype", [(np.float32, np.float32), (np.float64, np.float64),
                                                  (np.float64, np.float32)])
def test_shaded_march_bounded(ray_dtype, attr_dtype):
    dev = api.Device(0)
    field = Field.sphere(**workload.SPHERE)
    g = api.OccupancyGrid(128, Contraction.aabb(), dev=dev)
    for s in workload.grid_warmup_seeds(8, 5):
        g.update_field(field, 0.95, s)
    o, d = workload.orbit_rays(200, angle=0.4)
    rays, keep = _rays(dev, o, d, 0.2, 1.0, ray_dtype)
    _both(dev, g, rays, field, MarchConfig(5e-3, 1e-4, 1e-2), len(o), attr_dtype)
    # tiny step + no early stop: many rays overflow the 24-sample buffer -> fixup path
    _both(dev, g, rays, field, MarchConfig(1e-3, 0.0, 0.0), len(o), attr_dtype)


def test_shaded_march_growth_and_checker():
    dev = api.Device(0)
    con = Contraction.sphere((0.5, 0.5, 0.5), 0.5)
    field = Field.checker(0.2, 30.0, (0.9, 0.1, 0.2), (0.1, 0.8, 0.3))
    g = api.OccupancyGrid(48, con, dev=dev)
    for s in (1, 2):
        g.update_field(field, 0.95, s)
    rng = np.random.default_rng(3)
    d = rng.normal(size=(500, 3))
    d /= np.sqrt((d * d).sum(1))[:, None]
    o = np.tile([[0.5, 0.5, 0.5]], (500, 1))
    rays, keep = _rays(dev, o, d, 0.01, 20.0, np.float64)
    _both(dev, g, rays, field, MarchConfig(0.01, 1e-3, 1e-2, 256, 1.02), 500, np.float64)
    _render_both(dev, g, rays, field, MarchConfig(0.01, 1e-3, 1e-2, 256, 1.02), 500, np.float64)


def _render_both(dev, grid, rays, field, cfg, n, attr_dtype, time=0.0):
    """vmb_march_render_field == march_shaded -> render_forward, bit for bit."""
    a = api.march_device(dev, grid, rays, field, cfg, api.DevicePacked.allocate(dev, n, 8 * n + 1024))
    cap = a.capacity
    rgb_a, sig_a = dev.empty(cap * 3, attr_dtype), dev.empty(cap, attr_dtype)
    api.march_shaded_device(dev, grid, rays, field, cfg, a, rgb_a, sig_a, time)
    outs_a = [dev.empty(n * 3, attr_dtype), dev.empty(n, attr_dtype), dev.empty(n, attr_dtype)]
    api.render_forward_device(dev, a, rgb_a, sig_a, *outs_a)
    b = api.DevicePacked.allocate(dev, n, cap)
    rgb_b, sig_b = dev.empty(cap * 3, attr_dtype), dev.empty(cap, attr_dtype)
    outs_b = [dev.empty(n * 3, attr_dtype), dev.empty(n, attr_dtype), dev.empty(n, attr_dtype)]
    api.march_render_device(dev, grid, rays, field, cfg, b, rgb_b, sig_b, *outs_b, time=time)
    ha, hb = a.to_host(), b.to_host()
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(ha, k), getattr(hb, k)), k
    s = a.n_samples
    assert np.array_equal(rgb_a.numpy(3 * s), rgb_b.numpy(3 * s))
    assert np.array_equal(sig_a.numpy(s), sig_b.numpy(s))
    for x, y in zip(outs_a, outs_b):
        assert np.array_equal(x.numpy(), y.numpy())


@pytest.mark.parametrize("ray_dtype,attr_dtype", [(np.float32, np.float32), (np.float64, np.float64)])
def test_fused_forward_render(ray_dtype, attr_dtype):
    dev = api.Device(0)
    field = Field.sphere(center=(0.5, 0.5, 0.5), radius=0.2, sigma=200.0, rgb=(0.8, 0.25, 0.1))
    g = api.OccupancyGrid(128, Contraction.aabb(), dev=dev)
    for s in workload.grid_warmup_seeds(8, 5):
        g.update_field(field, 0.95, s)
    o, d = workload.orbit_rays(160, angle=2.0)
    rays, keep = _rays(dev, o, d, 0.2, 1.0, ray_dtype)
    _render_both(dev, g, rays, field, MarchConfig(5e-3, 1e-4, 1e-2), len(o), attr_dtype)
    # non-f32-representable sigma, long rays (overflow -> fixup composites), a box field
    box = Field.box((0.3, 0.2, 0.25), (0.7, 0.8, 0.75), 0.37, (0.3, 0.6, 0.9))
    gb = api.OccupancyGrid(64, Contraction.aabb(), 1e-3, dev=dev)
    gb.update_field(box, 0.95, 3)
    _render_both(dev, gb, rays, box, MarchConfig(2e-3, 0.0, 1e-4), len(o), attr_dtype)


def test_async_fused_forward_matches_sync():
    """vmb_march_render_field_async: same samples/attributes/outputs as the
    synchronous call, total on the device, errors deferred to vmb_march_check."""
    import ctypes as C
    from paper_2210_04847_b200._lib import VMB_F32 as F32, check
    dev = api.Device(0)
    L = dev.lib
    field = Field.sphere(**workload.SPHERE)
    g = api.OccupancyGrid(128, Contraction.aabb(), dev=dev)
    for s in workload.grid_warmup_seeds(8, 5):
        g.update_field(field, 0.95, s)
    o, d = workload.orbit_rays(96, angle=0.3)
    n = len(o)
    rays, keep = _rays(dev, o, d, 0.2, 1.0, np.float32)
    cfg = MarchConfig(5e-3, 1e-4, 1e-2)
    a = api.march_device(dev, g, rays, field, cfg, api.DevicePacked.allocate(dev, n, 8 * n + 1024))
    cap = a.capacity
    bufs = []
    for _ in range(2):
        bufs.append(dict(p=api.DevicePacked.allocate(dev, n, cap), rgb=dev.empty(3 * cap, np.float32),
                         sig=dev.empty(cap, np.float32),
                         out=[dev.empty(3 * n, np.float32), dev.empty(n, np.float32), dev.empty(n, np.float32)]))
    x, y = bufs
    api.march_render_device(dev, g, rays, field, cfg, x["p"], x["rgb"], x["sig"], *x["out"])
    nd = dev.zeros(1, np.uint64)
    smp = y["p"].samples_struct()
    check(L.vmb_march_render_field_async(dev.h, g.h, C.byref(rays), C.byref(field), C.byref(cfg), C.byref(smp),
                                         y["rgb"].ptr, y["sig"].ptr, y["out"][0].ptr, y["out"][1].ptr,
                                         y["out"][2].ptr, F32, 0.0, nd.ptr))
    check(L.vmb_march_check(dev.h))
    s = int(nd.numpy()[0])
    assert s == x["p"].n_samples > 0
    y["p"].n_samples = s
    hx, hy = x["p"].to_host(), y["p"].to_host()
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(hx, k), getattr(hy, k)), k
    assert np.array_equal(x["rgb"].numpy(3 * s), y["rgb"].numpy(3 * s))
    for u, v in zip(x["out"], y["out"]):
        assert np.array_equal(u.numpy(), v.numpy())
    # a negative density is recorded on the device and reported by vmb_march_check
    bad = Field.sphere(center=(0.5, 0.5, 0.5), radius=0.2, sigma=-1.0)
    check(L.vmb_march_render_field_async(dev.h, g.h, C.byref(rays), C.byref(bad), C.byref(cfg), C.byref(smp),
                                         y["rgb"].ptr, y["sig"].ptr, y["out"][0].ptr, y["out"][1].ptr,
                                         y["out"][2].ptr, F32, 0.0, nd.ptr))
    with pytest.raises(RuntimeError, match="negative density"):
        check(L.vmb_march_check(dev.h))
    check(L.vmb_march_check(dev.h))  # the record was reset


def test_step_is_bitwise_reproducible_and_chunk_independent():
    """The reference promises outputs independent of n_threads (test_ray_marching.cpp
    :180-199, test_rendering.cpp:350-371). Here: the fused step run twice gives the
    same bits (the walk's atomic chunk stealing does not leak into results), and
    marching the batch in two halves gives the same per-ray outputs."""
    dev = api.Device(0)
    field = Field.sphere(**workload.SPHERE)
    g = api.OccupancyGrid(128, Contraction.aabb(), dev=dev)
    for s in workload.grid_warmup_seeds(8, 5):
        g.update_field(field, 0.95, s)
    o, d = workload.orbit_rays(128, angle=0.7)
    n = len(o)
    cfg = MarchConfig(5e-3, 1e-4, 1e-2)

    def run(oo, dd):
        rays, keep = _rays(dev, oo, dd, 0.2, 1.0, np.float32)
        m = len(oo)
        p = api.march_device(dev, g, rays, field, cfg, api.DevicePacked.allocate(dev, m, 8 * m + 1024))
        cap = p.capacity
        rgb, sig = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)
        outs = [dev.empty(3 * m, np.float32), dev.empty(m, np.float32), dev.empty(m, np.float32)]
        api.march_render_device(dev, g, rays, field, cfg, p, rgb, sig, *outs)
        return p.to_host(), [x.numpy() for x in outs]

    (p1, o1), (p2, o2) = run(o, d), run(o, d)
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(p1, k), getattr(p2, k)), k
    for a, b in zip(o1, o2):
        assert np.array_equal(a, b)
    h = n // 2 + 17
    (pa, oa), (pb, ob) = run(o[:h], d[:h]), run(o[h:], d[h:])
    assert np.array_equal(np.concatenate([pa.counts, pb.counts]), p1.counts)
    assert np.array_equal(np.concatenate([pa.t_starts, pb.t_starts]), p1.t_starts)
    for a, b, full, w in zip(oa, ob, o1, (3, 1, 1)):
        assert np.array_equal(np.concatenate([a, b]), full)


def test_async_capacity_overflow_is_contained():
    """vmb_march_render_field_async with too small a sample capacity: the total on the
    device exceeds the capacity, samples beyond it are dropped, and the render
    kernels run on the truncated view ignore sample positions beyond n_samples
    instead of reading/writing past the buffers; rays wholly inside the capacity
    get the full run's gradients."""
    import ctypes as C
    from paper_2210_04847_b200._lib import VMB_F32 as F32, check
    dev = api.Device(0)
    L = dev.lib
    field = Field.sphere(**workload.SPHERE)
    g = api.OccupancyGrid(128, Contraction.aabb(), dev=dev)
    for s in workload.grid_warmup_seeds(8, 5):
        g.update_field(field, 0.95, s)
    o, d = workload.orbit_rays(64, angle=0.9)
    n = len(o)
    rays, keep = _rays(dev, o, d, 0.2, 1.0, np.float32)
    cfg = MarchConfig(5e-3, 1e-4, 1e-2)
    full = api.march_device(dev, g, rays, field, cfg, api.DevicePacked.allocate(dev, n, 16 * n))
    S = full.n_samples
    cap = S // 2
    rng = np.random.default_rng(3)
    ups = [dev.upload(rng.uniform(-1, 1, n * w).astype(np.float32)) for w in (3, 1, 1)]
    res = []
    for c in (full.capacity, cap):
        p = api.DevicePacked.allocate(dev, n, c)
        rgb, sig = dev.empty(3 * c, np.float32), dev.empty(c, np.float32)
        gr, gs = dev.empty(3 * c, np.float32), dev.empty(c, np.float32)
        outs = [dev.empty(3 * n, np.float32), dev.empty(n, np.float32), dev.empty(n, np.float32)]
        nd = dev.zeros(1, np.uint64)
        smp = p.samples_struct()
        check(L.vmb_march_render_field_async(dev.h, g.h, C.byref(rays), C.byref(field), C.byref(cfg), C.byref(smp),
                                             rgb.ptr, sig.ptr, outs[0].ptr, outs[1].ptr, outs[2].ptr, F32, 0.0,
                                             nd.ptr))
        p.n_samples = c
        api.render_backward_device(dev, p, rgb, sig, *ups, gr, gs)
        dev.sync()
        check(L.vmb_march_check(dev.h))
        assert int(nd.numpy()[0]) == S
        res.append((p.to_host() if c == full.capacity else None, gs.numpy(c), gr.numpy(3 * c)))
    hp = res[0][0]
    inside = hp.offsets.astype(np.int64) + hp.counts <= cap
    m = np.zeros(S, bool)
    for r in np.nonzero(inside)[0]:
        m[hp.offsets[r]:hp.offsets[r] + hp.counts[r]] = True
    mc = m[:cap]
    assert mc.sum() > 0
    assert np.array_equal(res[0][1][:cap][mc], res[1][1][mc])
    assert np.array_equal(res[0][2].reshape(-1, 3)[:cap][mc], res[1][2].reshape(-1, 3)[mc])


@pytest.mark.parametrize("ray_dtype,attr_dtype", [(np.float32, np.float32), (np.float64, np.float64),
                                                  (np.float32, np.float64)])
def test_march_render_long_ray_growth(ray_dtype, attr_dtype):
    """Growth lattices with > 16 kept samples per ray take k_shade_forward_win
    (shade + composite in one pass): bit for bit march_shaded -> render_forward."""
    dev = api.Device(0)
    con = Contraction.sphere((0.5, 0.5, 0.5), 0.5)
    field = Field.sphere(radius=0.3, sigma=40.0)
    g = api.OccupancyGrid(64, con, dev=dev)
    for s in (1, 2, 3):
        g.update_field(field, 0.95, s)
    rng = np.random.default_rng(5)
    d = rng.normal(size=(700, 3))
    d /= np.sqrt((d * d).sum(1))[:, None]
    o = np.tile([[0.5, 0.5, 0.55]], (700, 1))
    rays, keep = _rays(dev, o, d, 0.01, 100.0, ray_dtype)
    cfg = MarchConfig(1.6914558667664816e-3, 1e-4, 1e-2, 2048, 1.01)
    a = api.march_device(dev, g, rays, field, cfg, api.DevicePacked.allocate(dev, 700, 64 * 700))
    assert a.n_samples > 16 * 700
    _render_both(dev, g, rays, field, cfg, 700, attr_dtype)

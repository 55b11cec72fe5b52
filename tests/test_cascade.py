"""Multi-level (cascaded) occupancy grid and cone stepping — SURVEY §8a A19.

The reference has neither (non-goals); it has the single-level
OccupancyGrid and the geometric-growth walk (ray_marching.cpp:88-106). The cascade
is defined so that every level is a reference OccupancyGrid and the cascade query
is "the finest level whose domain contains the point decides" (include/vmb200.h,
vmb_march_ext). Pins:

  * levels = 1, no cone: vmb_march_cascade IS march() — bit-exact against the
    reference for the growth walk (A14) and the bounded lattice (A13);
  * each level is bit-exact to a reference OccupancyGrid built over the level's box
    (the grid tests), and the cascade query equals the composition of the
    reference's per-level queries;
  * cone stepping / stacked levels against the port's sequential restatement
    (oracle/vm_oracle.c vmo_march_cascade), bit-exact; widths follow
    dt = min(max(t cone_angle, step), max_step).
"""
import numpy as np
import pytest

from oracle import Oracle, available
from oracle import oracle as O

needs_ref = pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")
BASE = ((0.0, 0.0, 0.0), (1.0, 1.0, 1.0))


def level_box(level, lo=BASE[0], hi=BASE[1]):
    lo, hi = np.asarray(lo, float), np.asarray(hi, float)
    c, h = 0.5 * (lo + hi), 0.5 * (hi - lo)
    s = 2.0 ** level
    return tuple(c - h * s), tuple(c + h * s)


def port_cascade(orc, res, levels, field, seeds):
    grids = [orc.grid(res, O.Contraction.aabb(*level_box(l))) for l in range(levels)]
    for g in grids:
        for s in seeds:
            g.update_field(field, 0.95, s)
    return grids


def rays_inside(n, seed=0, origin=(0.5, 0.5, 0.85)):
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = np.tile(np.asarray(origin, float), (n, 1)) + rng.uniform(-0.05, 0.05, (n, 3))
    return o, d


BOX = O.Field.box((-2.0, 0.2, 0.1), (0.8, 0.9, 3.0), sigma=2.0, rgb=(0.2, 0.7, 0.3))
SEEDS = [11, 12, 13, 14]


def test_level_box_arithmetic():
    from paper_2210_04847_b200 import api
    from paper_2210_04847_b200._lib import Contraction, lib
    import ctypes as C
    base = Contraction.aabb((-0.25, 0.0, 0.5), (1.0, 2.0, 0.75))
    for level in range(8):
        out = Contraction()
        assert lib().vmb_cascade_level_box(C.byref(base), level, C.byref(out)) == 0
        lo, hi = level_box(level, (-0.25, 0.0, 0.5), (1.0, 2.0, 0.75))
        assert tuple(out.box_min) == lo and tuple(out.box_max) == hi
    out = Contraction()
    assert lib().vmb_cascade_level_box(C.byref(Contraction.sphere((0, 0, 0), 1.0)), 1, C.byref(out)) != 0
    assert api is not None


@needs_ref
def test_port_single_level_is_reference_march():
    """levels = 1, no cone: the cascade walk is the reference's march (A14 growth)."""
    ref, port = Oracle("ref"), Oracle("port")
    field = O.Field.sphere(radius=0.3, sigma=40.0)
    con = O.Contraction.sphere((0.5, 0.5, 0.5), 0.5)
    rg, pg = ref.grid(32, con), port.grid(32, con)
    for s in SEEDS:
        rg.update_field(field, 0.95, s)
        pg.update_field(field, 0.95, s)
    o, d = rays_inside(300, 1, (0.5, 0.5, 0.55))
    cfg = O.MarchConfig(1.6914558667664816e-3, 1e-4, 1e-2, 2048, 1.01)
    a = ref.march_field(o, d, 0.01, 100.0, rg, field, cfg)
    b = port.march_cascade(o, d, 0.01, 100.0, pg, [], field, cfg)
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.samples_emitted == b.samples_emitted


@needs_ref
def test_port_cascade_query_is_composition_of_reference_queries():
    ref, port = Oracle("ref"), Oracle("port")
    rgrids = port_cascade(ref, 16, 4, BOX, SEEDS)
    pgrids = port_cascade(port, 16, 4, BOX, SEEDS)
    for a, b in zip(rgrids, pgrids):
        assert np.array_equal(a.bits(), b.bits())
    rng = np.random.default_rng(3)
    pts = rng.uniform(-5, 6, (20000, 3))
    got = port.cascade_query(pgrids[0], pgrids[1:], pts)
    want = np.zeros(len(pts), bool)
    done = np.zeros(len(pts), bool)
    for level, g in enumerate(rgrids):
        lo, hi = level_box(level)
        inside = np.all((pts >= lo) & (pts <= hi), axis=1) & ~done
        want[inside] = g.query(pts[inside])
        done |= inside
    assert np.array_equal(got, want)


def test_port_cone_widths():
    port = Oracle("port")
    grids = port_cascade(port, 16, 4, BOX, SEEDS)
    o, d = rays_inside(200, 2)
    cfg = O.MarchConfig(2e-3, 1e-4, 0.0, 100000, 1.0)
    cone, max_step = 1.0 / 64, 0.05
    p = port.march_cascade(o, d, 0.01, 100.0, grids[0], grids[1:], BOX, cfg, cone, max_step)
    assert p.n_samples > 1000
    w = p.t_ends - p.t_starts
    want = np.minimum(np.maximum(p.t_starts * cone, 2e-3), max_step)
    last = p.t_ends == 100.0
    assert np.allclose(w[~last], want[~last], rtol=1e-12, atol=0)
    assert p.t_ends.max() > 1.5  # samples in the outer levels


# ------------------------------------------------------------------ device vs port
@pytest.fixture(scope="module")
def dev():
    from paper_2210_04847_b200 import api
    return api.Device(0)


def _device_cascade(dev, res, levels, field, seeds):
    from paper_2210_04847_b200 import api
    from paper_2210_04847_b200._lib import Contraction
    cas = api.Cascade(res, Contraction.aabb(*BASE), levels, dev=dev)
    for s in seeds:
        cas.update_field(field, 0.95, s)
    return cas


def _api_field(f):
    from paper_2210_04847_b200._lib import Field
    out = Field()
    for name, _ in O.Field._fields_:
        setattr(out, name, getattr(f, name))
    return out


class _DevRays:
    def __init__(self, dev, o, d, near, far):
        from paper_2210_04847_b200 import api
        self.keep = (dev.upload(np.asarray(o, float)), dev.upload(np.asarray(d, float)))
        self.rays = api.device_rays(dev, *self.keep, near, far)


def _march(dev, cas, o, d, near, far, field, cfg, cone=None, max_step=1e10, per_ray=64):
    from paper_2210_04847_b200 import api
    from paper_2210_04847_b200._lib import MarchConfig, MarchStats
    rays = _DevRays(dev, o, d, near, far)
    st = MarchStats()
    c = MarchConfig(cfg.step_size, cfg.early_stop_eps, cfg.alpha_thre, cfg.max_samples_per_ray,
                    cfg.unbounded_step_growth)
    out = api.DevicePacked.allocate(dev, len(o), per_ray * len(o))
    api.march_cascade_device(dev, cas, rays.rays, _api_field(field), c, out, cone, max_step, st)
    return out.to_host(), st


@pytest.mark.gpu
@pytest.mark.parametrize("levels,cone", [(4, 1.0 / 256), (4, None), (2, 1.0 / 64), (1, 1.0 / 128)])
def test_device_cascade_march_matches_port(dev, levels, cone):
    port = Oracle("port")
    pgrids = port_cascade(port, 32, levels, BOX, SEEDS)
    cas = _device_cascade(dev, 32, levels, _api_field(BOX), SEEDS)
    for g, q in zip(cas.grids, pgrids):
        assert np.array_equal(g.bits(), q.bits())
    o, d = rays_inside(4096, 5)
    cfg = O.MarchConfig(1.6914558667664816e-3, 1e-4, 1e-2, 4096, 1.0)
    max_step = 0.05 if cone else 1e10
    want = port.march_cascade(o, d, 0.01, 100.0, pgrids[0], pgrids[1:], BOX, cfg, cone, max_step)
    got, st = _march(dev, cas, o, d, 0.01, 100.0, BOX, cfg, cone, max_step)
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    assert st.samples_emitted == want.samples_emitted and st.samples_kept == want.samples_kept
    rng = np.random.default_rng(9)
    pts = rng.uniform(-5, 6, (50000, 3))
    assert np.array_equal(cas.query(pts), port.cascade_query(pgrids[0], pgrids[1:], pts))


@pytest.mark.gpu
@needs_ref
def test_device_single_level_cascade_is_reference_march(dev):
    """vmb_march_cascade with no stacked level and no cone = march(): the growth
    walk (sphere contraction) against the reference's own code."""
    from paper_2210_04847_b200 import api
    from paper_2210_04847_b200._lib import Contraction
    ref = Oracle("ref")
    field = O.Field.sphere(radius=0.3, sigma=40.0)
    rg = ref.grid(64, O.Contraction.sphere((0.5, 0.5, 0.5), 0.5))
    g = api.OccupancyGrid(64, Contraction.sphere((0.5, 0.5, 0.5), 0.5), dev=dev)
    for s in SEEDS:
        rg.update_field(field, 0.95, s)
        g.update_field(_api_field(field), 0.95, s)
    cas = api.Cascade.__new__(api.Cascade)
    cas.dev, cas.grids = dev, [g]
    import ctypes as C
    cas._arr = (C.c_void_p * 1)()
    o, d = rays_inside(2000, 7, (0.5, 0.5, 0.55))
    cfg = O.MarchConfig(1.6914558667664816e-3, 1e-4, 1e-2, 2048, 1.01)
    want = ref.march_field(o, d, 0.01, 100.0, rg, field, cfg)
    got, st = _march(dev, cas, o, d, 0.01, 100.0, field, cfg)
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    assert st.samples_emitted == want.samples_emitted


@pytest.mark.gpu
def test_device_cascade_render_matches_port(dev):
    from paper_2210_04847_b200 import api
    from paper_2210_04847_b200._lib import MarchConfig
    port = Oracle("port")
    pgrids = port_cascade(port, 32, 4, BOX, SEEDS)
    cas = _device_cascade(dev, 32, 4, _api_field(BOX), SEEDS)
    o, d = rays_inside(2048, 8)
    cfg = O.MarchConfig(1.6914558667664816e-3, 1e-4, 1e-2, 4096, 1.0)
    want = port.march_cascade(o, d, 0.01, 100.0, pgrids[0], pgrids[1:], BOX, cfg, 1 / 256, 0.05)
    rgb, sig = port.shade(o, d, want, BOX)
    col, op, dep = port.render_forward(want, rgb, sig)
    rays = _DevRays(dev, o, d, 0.01, 100.0)
    n = len(o)
    out = api.DevicePacked.allocate(dev, n, 2 * want.n_samples + 1024)
    cap = out.capacity
    drgb, dsig = dev.empty(3 * cap, np.float64), dev.empty(cap, np.float64)
    outs = [dev.empty(3 * n, np.float64), dev.empty(n, np.float64), dev.empty(n, np.float64)]
    api.march_render_cascade_device(dev, cas, rays.rays, _api_field(BOX), MarchConfig(*[getattr(cfg, k) for k in (
        "step_size", "early_stop_eps", "alpha_thre", "max_samples_per_ray", "unbounded_step_growth")]), out,
        drgb, dsig, *outs, cone_angle=1 / 256, max_step=0.05)
    got = out.to_host()
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    s = got.n_samples
    assert np.array_equal(drgb.numpy(3 * s).reshape(-1, 3), rgb)
    assert np.array_equal(dsig.numpy(s), sig)
    for a, b in zip(outs, (col.ravel(), op, dep)):
        assert np.allclose(a.numpy(), b, rtol=1e-12, atol=1e-14)


@pytest.mark.gpu
def test_cascade_errors(dev):
    from paper_2210_04847_b200 import api
    from paper_2210_04847_b200._lib import Contraction, MarchConfig
    cas = _device_cascade(dev, 16, 3, _api_field(BOX), SEEDS[:1])
    o, d = rays_inside(8, 1)
    rays = _DevRays(dev, o, d, 0.01, 100.0)
    out = api.DevicePacked.allocate(dev, 8, 1024)
    sph = api.Cascade.__new__(api.Cascade)  # growth applies to a sphere-contracted level 0 only
    sph.dev = dev
    sph.grids = [api.OccupancyGrid(16, Contraction.sphere((0.5, 0.5, 0.5), 0.5), dev=dev)]
    import ctypes as C
    sph._arr = (C.c_void_p * 1)()
    with pytest.raises(ValueError, match="cone stepping and unbounded_step_growth"):
        api.march_cascade_device(dev, sph, rays.rays, _api_field(BOX), MarchConfig(1e-2, 1e-4, 1e-2, 64, 1.01),
                                 out, 0.01)
    with pytest.raises(ValueError, match="max_step must be >= step_size"):
        api.march_cascade_device(dev, cas, rays.rays, _api_field(BOX), MarchConfig(1e-2, 1e-4, 1e-2, 64, 1.0),
                                 out, 0.01, 1e-3)
    bad = api.Cascade.__new__(api.Cascade)
    bad.dev = dev
    bad.grids = [cas.grids[1], cas.grids[0]]  # level 1 below level 0: not nested
    import ctypes as C
    bad._arr = (C.c_void_p * 1)(cas.grids[0].h.value)
    with pytest.raises(ValueError, match="strictly contain"):
        api.march_cascade_device(dev, bad, rays.rays, _api_field(BOX), MarchConfig(1e-2, 1e-4, 1e-2, 64, 1.0),
                                 out, 0.01)
    assert Contraction is not None


@pytest.mark.gpu
def test_device_cascade_long_rays_past_the_slab_match_port(dev):
    """Long-ray walks pack in one walk (a per-ray slab of 256 intervals, then a fill of
    the rays above it): rays with no transmittance cut through a dense field keep
    hundreds of samples each, so both the slab gather and the overflow fill run."""
    port = Oracle("port")
    dense = O.Field.box((-9.0, -9.0, -9.0), (9.0, 9.0, 1.0), sigma=20.0, rgb=(0.5, 0.5, 0.5))
    pgrids = port_cascade(port, 32, 3, dense, SEEDS)
    cas = _device_cascade(dev, 32, 3, _api_field(dense), SEEDS)
    o, d = rays_inside(1024, 21)
    cfg = O.MarchConfig(1.6914558667664816e-3, 0.0, 1e-4, 100000, 1.0)
    want = port.march_cascade(o, d, 0.01, 100.0, pgrids[0], pgrids[1:], dense, cfg, 1.0 / 256, 0.02)
    got, st = _march(dev, cas, o, d, 0.01, 100.0, dense, cfg, 1.0 / 256, 0.02, per_ray=int(want.counts.max()) + 1)
    assert want.counts.max() > 256 and (want.counts <= 256).any()
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    assert st.samples_emitted == want.samples_emitted and st.samples_kept == want.samples_kept

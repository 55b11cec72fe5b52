"""Parity of the CUDA path (via the C ABI) with the CPU oracle.

Bit-exact: grid bits/cache, sample counts, offsets (packed_info), ray_indices and
t_starts/t_ends. Rendering outputs and gradients: rtol 1e-5 with an absolute floor
of 1e-8 (close_rel of proj/tests/unit/test_rendering.cpp:67-69); in practice the
fp64 kernels agree to ~1e-15.
"""
import os
import tempfile

import numpy as np
import pytest

from oracle import Oracle, available
from oracle import oracle as O
from paper_2210_04847_b200 import api, workload
from paper_2210_04847_b200._lib import Contraction, Field, MarchConfig, MarchStats

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RTOL, ATOL = 1e-5, 1e-8


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


def ocon(c: Contraction):
    o = O.Contraction()
    for name, _ in Contraction._fields_:
        setattr(o, name, getattr(c, name))
    return o


def ocfg(c: MarchConfig):
    return O.MarchConfig(c.step_size, c.early_stop_eps, c.alpha_thre, c.max_samples_per_ray,
                         c.unbounded_step_growth)


def close(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    assert a.shape == b.shape
    tol = np.maximum(RTOL * np.maximum(np.abs(a), np.abs(b)), ATOL)
    bad = np.abs(a - b) > tol
    assert not bad.any(), f"{bad.sum()} mismatches, worst {np.abs(a - b).max()}"


def same_packed(p, q):
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(p, k), getattr(q, k)), k


def both_grids(dev, orc, res, con, field, seeds, timestamps=(0.0,), thr=1e-2, init=0.0):
    g = api.OccupancyGrid(res, con, thr, 0.0, init, dev=dev)
    og = orc.grid(res, ocon(con), thr, 0.0, init)
    for s in seeds:
        g.update_field(field, 0.95, s, timestamps)
        og.update_field(ofield(field), 0.95, s, timestamps)
    return g, og


# ------------------------------------------------------------------ occupancy grid
@pytest.mark.parametrize("res", [128, 256])
def test_grid_update_bit_exact_config5(dev, orc, res):
    field = Field.sphere(**workload.SPHERE)
    g, og = both_grids(dev, orc, res, Contraction.aabb(), field, workload.grid_warmup_seeds(16, 5))
    assert np.array_equal(g.bits(), og.bits())
    assert np.array_equal(g.density_cache(), og.cache())
    assert g.occupied_fraction() == og.info()["occupied_fraction"]


def test_grid_golden_config1(dev):
    z = np.load(os.path.join(G, "c1.npz"))
    field = Field.sphere(**workload.SPHERE)
    g = api.OccupancyGrid(128, Contraction.aabb(), dev=dev)
    for s in workload.grid_warmup_seeds(16, 5):
        g.update_field(field, 0.95, s)
    assert np.array_equal(g.packed_bits(), z["bits"])
    assert np.array_equal(g.density_cache().astype(np.float32), z["cache"])


@pytest.mark.parametrize("con", [Contraction.sphere((0.5, 0.5, 0.5), 0.5),
                                 Contraction.aabb((-0.5, 0.0, 0.0), (1.5, 1.0, 2.0)),
                                 Contraction.aabb((0.1, 0.2, 0.3), (0.9, 0.7, 1.0))])
def test_grid_contractions_and_time(dev, orc, con):
    field = Field.sphere(center=(0.3, 0.5, 0.5), radius=0.25, sigma=60.0, velocity=(0.3, 0.0, 0.1))
    g, og = both_grids(dev, orc, 48, con, field, [1, 2, None, 3], timestamps=(0.0, 0.5, 1.0))
    assert np.array_equal(g.bits(), og.bits())
    assert np.array_equal(g.density_cache(), og.cache())
    pts = np.random.default_rng(0).uniform(-0.6, 1.6, (20000, 3))
    assert np.array_equal(g.query(pts), og.query(pts))


def test_grid_callback_path_and_errors(dev, orc):
    def fn(p, t):
        return 30.0 * (np.sin(7 * p[:, 0] + t) > 0.3)

    g = api.OccupancyGrid(24, Contraction.sphere((0.5, 0.5, 0.5), 0.6), dev=dev)
    og = orc.grid(24, O.Contraction.sphere((0.5, 0.5, 0.5), 0.6))
    g.update_over_time(fn, (0.0, 2.0), 0.9, 11)
    og.update_callback(fn, 0.9, 11, (0.0, 2.0))
    assert np.array_equal(g.density_cache(), og.cache()) and np.array_equal(g.bits(), og.bits())
    bad = api.OccupancyGrid(4, Contraction.aabb(), dev=dev)
    with pytest.raises(RuntimeError, match=r"^occupancy grid: invalid density at cell \(1,1,0\)$"):
        bad.update(lambda p: np.where(np.arange(len(p)) == 5, -2.0, 1.0), 0.95)
    with pytest.raises(ValueError, match="timestamps must be non-empty"):
        bad.update_over_time(fn, [], 0.95)
    with pytest.raises(ValueError, match="non-finite coordinate"):
        bad.query([[np.nan, 0, 0]])


def test_grid_invalid_sigma_field_names_first_cell(dev, orc):
    f = Field.box((0.3, 0.3, 0.3), (0.6, 0.6, 0.6), sigma=-1.0)
    g = api.OccupancyGrid(16, Contraction.aabb(), dev=dev)
    og = orc.grid(16, O.Contraction.aabb())
    with pytest.raises(O.OracleError) as e:
        og.update_field(ofield(f), 0.95, 7)
    with pytest.raises(RuntimeError) as e2:
        g.update_field(f, 0.95, 7)
    assert str(e2.value) == e.value.msg
    assert np.array_equal(g.density_cache(), np.zeros(16 ** 3))  # grid untouched


def test_grid_seed_fraction_and_ogrd(dev, orc):
    rng = np.random.default_rng(3)
    mask = (rng.uniform(size=32 ** 3) < 0.3).astype(np.uint8)
    g = api.OccupancyGrid(32, Contraction.aabb(), dev=dev)
    og = orc.grid(32, O.Contraction.aabb())
    g.seed_mask(mask)
    og.seed_mask(mask)
    assert np.array_equal(g.bits(), og.bits()) and np.array_equal(g.density_cache(), og.cache())
    with tempfile.TemporaryDirectory() as tmp:
        gs = api.OccupancyGrid(16, Contraction.sphere((0.5, 0.5, 0.5), 0.75), 2e-2, 0.001, dev=dev)
        gs.update_field(Field.sphere(radius=0.4, sigma=60.0), 0.95, 1234)
        a = os.path.join(tmp, "a.ogrd")
        gs.save(a)
        lo = orc.grid_load(a)  # the reference reads our file
        b = os.path.join(tmp, "b.ogrd")
        lo.save(b)
        assert open(a, "rb").read() == open(b, "rb").read()
        lg = api.OccupancyGrid.load(b, dev)
        assert np.array_equal(lg.bits(), lo.bits()) and np.array_equal(lg.density_cache(), lo.cache())


# ------------------------------------------------------------------ marching
def test_march_golden_config1(dev):
    z = np.load(os.path.join(G, "c1.npz"))
    field = Field.sphere(**workload.SPHERE)
    g = api.OccupancyGrid(128, Contraction.aabb(), dev=dev)
    for s in workload.grid_warmup_seeds(16, 5):
        g.update_field(field, 0.95, s)
    o, d = workload.orbit_rays(64)
    st = MarchStats()
    p = api.march(api.RayBatch.create(o, d, 0.2, 1.0, dev), g, field, MarchConfig(5e-3, 1e-4, 1e-2),
                  stats=st)
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(p, k), z[k]), k
    assert st.samples_emitted == 107555 and st.samples_kept == 19362


@pytest.mark.parametrize("cfg", [MarchConfig(5e-3, 1e-4, 1e-2), MarchConfig(1.6914558667664816e-3),
                                 MarchConfig(0.011, 0.0, 0.0), MarchConfig(5e-3, 0.5, 0.3),
                                 MarchConfig(0.003, 1e-3, 0.0, max_samples_per_ray=7)])
def test_march_field_bit_exact(dev, orc, cfg):
    field = Field.sphere(**workload.SPHERE)
    g, og = both_grids(dev, orc, 64, Contraction.aabb(), field, workload.grid_warmup_seeds(6, 5))
    o, d = workload.orbit_rays(96, angle=0.3)
    rng = np.random.default_rng(1)
    ro = rng.uniform(-0.2, 1.2, (3000, 3))
    rd = rng.normal(size=(3000, 3))
    rd /= np.sqrt((rd * rd).sum(1))[:, None]
    for (oo, dd, near, far) in [(o, d, 0.2, 1.0), (ro, rd, 0.0, 1.7)]:
        st = MarchStats()
        p = api.march(api.RayBatch.create(oo, dd, near, far, dev), g, field, cfg, stats=st)
        q = orc.march_field(oo, dd, near, far, og, ofield(field), ocfg(cfg), 4)
        same_packed(p, q)
        assert st.samples_emitted == q.samples_emitted


def test_march_other_fields_and_boxes(dev, orc):
    con = Contraction.aabb((-1.0, -0.5, 0.0), (1.0, 1.5, 3.0))  # non power-of-two sizes
    for field in (Field.box((-0.5, 0.0, 0.5), (0.5, 1.0, 2.0), 30.0, (0.2, 0.3, 0.4)),
                  Field.checker(0.3, 4.0, (0.9, 0.1, 0.2), (0.1, 0.8, 0.3))):
        g, og = both_grids(dev, orc, 40, con, field, [5, 6])
        rng = np.random.default_rng(2)
        ro = rng.uniform(-1.2, 1.2, (2000, 3))
        rd = rng.normal(size=(2000, 3))
        rd /= np.sqrt((rd * rd).sum(1))[:, None]
        cfg = MarchConfig(0.02, 1e-3, 1e-2)
        p = api.march(api.RayBatch.create(ro, rd, 0.0, 4.0, dev), g, field, cfg)
        same_packed(p, orc.march_field(ro, rd, 0.0, 4.0, og, ofield(field), ocfg(cfg), 4))


def test_march_growth_golden(dev):
    z = np.load(os.path.join(G, "growth.npz"))
    con = Contraction.sphere((0.5, 0.5, 0.5), 0.5)
    field = Field.sphere(radius=0.3, sigma=40.0)
    g = api.OccupancyGrid(64, con, dev=dev)
    for s in (1, 2, 3):
        g.update_field(field, 0.95, s)
    assert np.array_equal(g.packed_bits(), z["bits"])
    cfg = MarchConfig(1.6914558667664816e-3, 1e-4, 1e-2, 2048, 1.01)
    st = MarchStats()
    p = api.march(api.RayBatch.create(z["origins"], z["dirs"], 0.01, 100.0, dev), g, field, cfg, stats=st)
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(p, k), z[k]), k
    assert st.samples_emitted == z["emitted"]


def test_march_callback_and_errors(dev, orc):
    field = Field.sphere(**workload.SPHERE)
    g, og = both_grids(dev, orc, 32, Contraction.aabb(), field, [1, 2])
    o, d = workload.orbit_rays(24)

    def sig(ts, te, idx):
        mid = 0.5 * (ts + te)
        return 50.0 * (0.5 + 0.5 * np.sin(20 * mid))

    cfg = MarchConfig(0.01, 1e-3, 0.0)
    st = MarchStats()
    p = api.march(api.RayBatch.create(o, d, 0.2, 1.0, dev), g, sig, cfg, stats=st)
    q = orc.march_callback(o, d, 0.2, 1.0, og, sig, ocfg(cfg))
    same_packed(p, q)
    assert st.samples_emitted == q.samples_emitted
    full = api.OccupancyGrid(8, Contraction.aabb(), 1e-2, 0.0, 1e6, dev=dev)
    rays = api.RayBatch.create([[0.0, 0.5, 0.5]], [[1.0, 0.0, 0.0]], 0.2, 1.0, dev)
    with pytest.raises(RuntimeError, match=r"^marching: non-finite density at ray 0 sample 7$"):
        api.march(rays, full, lambda ts, te, i: np.r_[np.ones(len(ts) - 1), np.nan], MarchConfig(0.1))
    with pytest.raises(RuntimeError, match=r"^marching: sigma_fn returned 9 values for 8 samples$"):
        api.march(rays, full, lambda ts, te, i: np.ones(len(ts) + 1), MarchConfig(0.1))
    with pytest.raises(RuntimeError, match=r"^marching: negative density at ray 0 sample 3$"):
        api.march(rays, full, lambda ts, te, i: np.where(np.arange(len(ts)) == 3, -1.0, 0.5), MarchConfig(0.1))
    def second_ray_negative(ts, te, idx):
        return np.full(len(ts), -1.0 if idx[0] == 1 else 0.5)

    two = api.RayBatch.create([[0.0, 0.5, 0.5]] * 2, [[1.0, 0.0, 0.0]] * 2, 0.2, 1.0, dev)
    with pytest.raises(RuntimeError, match=r"^marching: negative density at ray 1 sample 0$"):
        api.march(two, full, second_ray_negative, MarchConfig(0.1))
    with pytest.raises(RuntimeError, match=r"^marching: negative density at ray 0 sample 0$"):
        api.march(rays, full, Field.box((0, 0, 0), (1, 1, 1), -1.0), MarchConfig(0.1))
    with pytest.raises(ValueError, match="step_size must be > 0"):
        api.march(rays, full, field, MarchConfig(0.0))
    with pytest.raises(ValueError, match="non-unit direction at index 1"):
        api.RayBatch.create([[0, 0, 0]] * 2, [[1, 0, 0], [1, 1, 0]], 0.2, 1.0, dev)


def test_march_uniform(dev, orc):
    rng = np.random.default_rng(7)
    o = rng.uniform(0, 1, (64, 3))
    d = rng.normal(size=(64, 3))
    d /= np.sqrt((d * d).sum(1))[:, None]
    for near, far, step in [(0.2, 1.0, 0.1), (0.2, 0.25, 0.1), (0.0, 3.0, 0.0137)]:
        p = api.march_uniform(api.RayBatch.create(o, d, near, far, dev), MarchConfig(step), dev)
        same_packed(p, orc.march_uniform(o, d, near, far, O.MarchConfig(step)))
    empty = api.march_uniform(api.RayBatch.create(np.zeros((0, 3)), np.zeros((0, 3)), 0.2, 1.0, dev),
                              MarchConfig(0.1), dev)
    assert empty.n_rays == 0 and empty.n_samples == 0


def test_march_large_batch_matches_reference(dev, orc):
    """2^20 rays of the bench camera (config 4 size) against the oracle."""
    field = Field.sphere(**workload.SPHERE)
    g, og = both_grids(dev, orc, 128, Contraction.aabb(), field, workload.grid_warmup_seeds(16, 5))
    o, d = workload.orbit_rays(1024)
    cfg = MarchConfig(5e-3, 1e-4, 1e-2)
    p = api.march(api.RayBatch.create(o, d, 0.2, 1.0, dev), g, field, cfg)
    q = orc.march_field(o, d, 0.2, 1.0, og, ofield(field), ocfg(cfg), os.cpu_count() or 1)
    same_packed(p, q)
    assert p.n_samples == 4951339


# ------------------------------------------------------------------ packing
def test_pack_and_validate(dev, orc):
    off, idx = api.pack([2, 0, 3], dev)
    assert list(off) == [0, 2, 2] and list(idx) == [0, 0, 2, 2, 2]
    off, idx = api.pack([], dev)
    assert len(off) == 0 and len(idx) == 0
    rng = np.random.default_rng(4)
    c = rng.integers(0, 9, 100000).astype(np.uint32)
    o1, i1 = api.pack(c, dev)
    o2, i2 = orc.pack(c)
    assert np.array_equal(o1, o2) and np.array_equal(i1, i2)
    with pytest.raises(ValueError, match="sample count exceeds 32-bit index range"):
        api.pack(np.array([0x80000000, 0x80000001], np.uint32), dev)
    counts = np.array([2, 0, 3], np.uint32)
    off, idx = orc.pack(counts)
    ts = np.array([0.1, 0.3, 0.0, 0.2, 0.5])
    te = np.array([0.2, 0.4, 0.1, 0.3, 0.6])
    cases = [(off, counts, ts, te, idx), (np.array([0, 1, 2], np.uint32), counts, ts, te, idx),
             (off, counts, ts, np.where(np.arange(5) == 3, 0.2, te), idx),
             (off, counts, np.array([0.1, 0.3, 0.3, 0.2, 0.5]), te, idx),
             (off, counts, ts, np.array([0.2, 0.4, 0.1, 0.35, 0.6]), idx),
             (off, counts, ts, te, np.array([0, 0, 2, 1, 2], np.uint32)),
             (off, counts, ts[:4], te, idx)]
    for c_ in cases:
        assert api.validate(api.PackedSamples(*c_), dev) == orc.validate(*c_)


# ------------------------------------------------------------------ rendering
def test_render_golden_instances(dev):
    z = np.load(os.path.join(G, "render.npz"))
    for i in range(60):
        k = lambda n: z[f"{i}_{n}"]  # noqa: E731
        p = api.PackedSamples(k("offsets"), k("counts"), k("t_starts"), k("t_ends"),
                              np.repeat(np.arange(len(k("counts")), dtype=np.uint32), k("counts")))
        close(api.transmittance(p, k("sigmas"), dev), k("trans"))
        c, o, d = api.render_forward(p, k("rgbs"), k("sigmas"), dev=dev)
        close(c, k("color")), close(o, k("opacity")), close(d, k("depth"))
        dr, ds = api.render_backward(p, k("rgbs"), k("sigmas"), k("d_color"), k("d_opacity"),
                                     k("d_depth"), dev=dev)
        close(dr, k("d_rgbs")), close(ds, k("d_sigmas"))
        close(api.render_attribute(p, k("sigmas"), k("values"), 2, dev), k("attr"))


def _instance(rng, n_rays, max_per_ray, contiguous=True):
    counts = rng.integers(0, max_per_ray + 1, n_rays).astype(np.uint32)
    offsets = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint32)
    s = int(counts.sum())
    ts = np.empty(s)
    te = np.empty(s)
    for r in range(n_rays):
        b, c = offsets[r], counts[r]
        w = rng.uniform(0.01, 0.2, c)
        t0 = rng.uniform(0, 0.5) + np.concatenate([[0], np.cumsum(w)[:-1]])
        ts[b:b + c], te[b:b + c] = t0, t0 + w
    p = O.Packed(offsets, counts, ts, te, np.repeat(np.arange(n_rays, dtype=np.uint32), counts))
    if not contiguous:  # reverse the ray order of the storage: offsets no longer ascending
        perm = np.arange(n_rays)[::-1]
        new_off = np.zeros(n_rays, np.uint32)
        ts2, te2, at = np.empty(s), np.empty(s), 0
        for r in perm:
            b, c = offsets[r], counts[r]
            ts2[at:at + c], te2[at:at + c] = ts[b:b + c], te[b:b + c]
            new_off[r] = at
            at += c
        p = O.Packed(new_off, counts, ts2, te2, np.zeros(s, np.uint32))
    return p, rng.uniform(0, 1, (s, 3)), rng.uniform(0, 8, s)


@pytest.mark.parametrize("n_rays,max_per_ray,contiguous",
                         [(3000, 12, True), (500, 300, True), (257, 40, False), (64, 2048, True),
                          (2000, 100, True)])  # rays around the half-tile cut (64 f32, 32 f64) in every warp
def test_render_paths_vs_oracle(dev, orc, n_rays, max_per_ray, contiguous):
    rng = np.random.default_rng(n_rays)
    p, rgb, sig = _instance(rng, n_rays, max_per_ray, contiguous)
    n = p.n_rays
    dc, do, dd = rng.uniform(-1, 1, (n, 3)), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    ap = api.PackedSamples(p.offsets, p.counts, p.t_starts, p.t_ends, p.ray_indices)
    for dtype in (np.float64, np.float32):
        r32 = rgb.astype(dtype).astype(np.float64)
        s32 = sig.astype(dtype).astype(np.float64)
        ref_f = orc.render_forward(p, r32, s32)
        ref_b = orc.render_backward(p, r32, s32, dc.astype(dtype), do.astype(dtype), dd.astype(dtype))
        got_f = api.render_forward(ap, r32, s32, dev=dev, dtype=dtype)
        got_b = api.render_backward(ap, r32, s32, dc, do, dd, dev=dev, dtype=dtype)
        for a, b in zip(got_f, ref_f):
            close(a, b)
        for a, b in zip(got_b, ref_b):
            close(a, b)
    close(api.transmittance(ap, sig, dev), orc.transmittance(p, sig))


def test_render_pack_with_gaps_zero_fills(dev, orc):
    """Rays covering only part of [0, n_samples): gaps between rays and a trailing
    gap. The reference zero-initialises the per-sample outputs (rendering.cpp:22,
    78-79), so the uncovered samples must come back 0, not stale memory."""
    rng = np.random.default_rng(11)
    p, rgb, sig = _instance(rng, 400, 20, True)
    n, s = p.n_rays, len(p.t_starts)
    gap = rng.integers(0, 3, n).astype(np.uint32)  # holes before each ray
    new_off = (p.offsets + np.cumsum(gap)).astype(np.uint32)
    tot = int(new_off[-1] + p.counts[-1]) + 7  # + a trailing gap
    ts, te = np.zeros(tot), np.zeros(tot)
    for r in range(n):
        b, c, nb = p.offsets[r], p.counts[r], new_off[r]
        ts[nb:nb + c], te[nb:nb + c] = p.t_starts[b:b + c], p.t_ends[b:b + c]
    covered = np.zeros(tot, bool)
    for r in range(n):
        covered[new_off[r]:new_off[r] + p.counts[r]] = True
    te[~covered] = ts[~covered] + 0.05
    rgb2, sig2 = rng.uniform(0, 1, (tot, 3)), rng.uniform(0, 8, tot)
    q = O.Packed(new_off, p.counts, ts, te, np.zeros(tot, np.uint32))
    aq = api.PackedSamples(new_off, p.counts, ts, te, np.zeros(tot, np.uint32))
    dc, do, dd = rng.uniform(-1, 1, (n, 3)), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    for _ in range(2):  # the second call reuses freed device memory holding the first's outputs
        got = api.render_backward(aq, rgb2, sig2, dc, do, dd, dev=dev)
        ref = orc.render_backward(q, rgb2, sig2, dc, do, dd)
        for a, b in zip(got, ref):
            close(a, b)
        assert not np.asarray(got[1])[~covered].any() and not np.asarray(got[0])[~covered].any()
        tr = api.transmittance(aq, sig2, dev)
        close(tr, orc.transmittance(q, sig2))
        assert not np.asarray(tr)[~covered].any()


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_render_forward_long_ray_kernel_bit_identical(dev, orc, dtype):
    """Batches averaging > 16 samples per ray take k_forward_win (staged windows,
    lane per ray); the same rays padded with empty rays (average below 16) take
    the tile kernel: the outputs must agree bit for bit (same expressions, same
    order, rendering.cpp:47-58)."""
    rng = np.random.default_rng(7)
    p, rgb, sig = _instance(rng, 300, 200, True)
    n, s = p.n_rays, len(p.t_starts)
    assert s > 16 * n
    r32 = rgb.astype(dtype).astype(np.float64)
    s32 = sig.astype(dtype).astype(np.float64)
    pad = 40 * n
    off = np.concatenate([p.offsets, np.full(pad, s, np.uint32)]).astype(np.uint32)
    cnt = np.concatenate([p.counts, np.zeros(pad, np.uint32)]).astype(np.uint32)
    a = api.PackedSamples(p.offsets, p.counts, p.t_starts, p.t_ends, p.ray_indices)
    b = api.PackedSamples(off, cnt, p.t_starts, p.t_ends, p.ray_indices)
    fa = api.render_forward(a, r32, s32, dev=dev, dtype=dtype)
    fb = api.render_forward(b, r32, s32, dev=dev, dtype=dtype)
    for x, y in zip(fa, fb):
        assert np.array_equal(np.asarray(x), np.asarray(y)[:n])
    for x, y in zip(fa, orc.render_forward(p, r32, s32)):
        close(x, y)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("contiguous", [True, False])
def test_render_backward_long_rays_vs_reference(dev, orc, dtype, contiguous):
    """Rays longer than a tile go to k_backward_long (one warp per ray: product scan
    for T, suffix of w v accumulated from the ray's end); warps whose rays are not
    stored contiguously run the same per-ray path."""
    rng = np.random.default_rng(11)
    p, rgb, sig = _instance(rng, 300, 400, contiguous)
    n = p.n_rays
    r32 = rgb.astype(dtype).astype(np.float64)
    s32 = sig.astype(dtype).astype(np.float64)
    dc, do, dd = rng.uniform(-1, 1, (n, 3)), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    ap = api.PackedSamples(p.offsets, p.counts, p.t_starts, p.t_ends, p.ray_indices)
    got = api.render_backward(ap, r32, s32, dc, do, dd, dev=dev, dtype=dtype)
    for x, y in zip(got, orc.render_backward(p, r32, s32, dc.astype(dtype), do.astype(dtype), dd.astype(dtype))):
        close(x, y)


@pytest.mark.parametrize("count", [3000, 6000])
def test_render_backward_long_dense_ray_tail_relative_error(dev, orc, count):
    """One long, dense ray with no transmittance cut (a user-built pack): T falls to
    ~1e-150 and the tail's d_sigma is tiny. The suffix is accumulated from the
    ray's end (rendering.cpp:99-108), never as total - prefix, so every sample's
    d_sigma keeps its relative accuracy (count 6000: more tiles than one
    super-block of carried transmittances)."""
    rng = np.random.default_rng(count)
    w = np.full(count, 0.01)
    ts = 0.2 + np.concatenate([[0.0], np.cumsum(w)[:-1]])
    te = ts + w
    sig = rng.uniform(5.0, 15.0, count)
    rgb = rng.uniform(0, 1, (count, 3))
    p = O.Packed(np.array([0], np.uint32), np.array([count], np.uint32), ts, te, np.zeros(count, np.uint32))
    ap = api.PackedSamples(p.offsets, p.counts, p.t_starts, p.t_ends, p.ray_indices)
    dc, do, dd = np.array([[0.3, -0.7, 0.5]]), np.array([0.25]), np.array([-0.4])
    got_rgb, got_sig = api.render_backward(ap, rgb, sig, dc, do, dd, dev=dev)
    ref_rgb, ref_sig = orc.render_backward(p, rgb, sig, dc, do, dd)
    nz = ref_sig != 0
    assert nz.sum() > count // 2
    rel = np.abs(got_sig[nz] - ref_sig[nz]) / np.abs(ref_sig[nz])
    assert rel.max() < 1e-9, rel.max()
    close(got_rgb, ref_rgb)


def test_render_closed_forms(dev):
    p = api.PackedSamples(np.array([0], np.uint32), np.array([2], np.uint32), np.array([0.0, 1.0]),
                          np.array([1.0, 2.0]), np.array([0, 0], np.uint32))
    c, o, _ = api.render_forward(p, [[1, 0, 0], [0, 1, 0]], [np.log(2.0)] * 2, dev=dev)
    assert abs(c[0, 0] - 0.5) < 1e-12 and abs(c[0, 1] - 0.25) < 1e-12 and c[0, 2] == 0.0
    assert abs(o[0] - 0.75) < 1e-12
    t = api.transmittance(p, [np.log(2.0), 3.0], dev)
    assert t[0] == 1.0 and abs(t[1] - 0.5) < 1e-12
    with pytest.raises(ValueError, match="attribute length mismatch"):
        api.render_forward(p, [[1, 1, 1]], [1.0], dev=dev)
    z = api.PackedSamples(np.array([0, 0], np.uint32), np.array([0, 0], np.uint32))
    _, o, _ = api.render_forward(z, np.zeros((0, 3)), np.zeros(0), dev=dev)
    assert list(o) == [0.0, 0.0]


# ------------------------------------------------------------------ skipping stress tests
def _stress_rays(rng, n):
    o = rng.uniform(-0.6, 1.6, (n, 3))
    d = rng.normal(size=(n, 3))
    k = n // 4
    # axis-aligned and single-zero-component directions; origins on cell faces
    d[:k] = np.eye(3)[rng.integers(0, 3, k)] * rng.choice([-1.0, 1.0], (k, 1))
    d[k:2 * k, rng.integers(0, 3)] = 0.0
    o[2 * k:3 * k] = np.round(o[2 * k:3 * k] * 64) / 64
    d /= np.sqrt((d * d).sum(1))[:, None]
    return o, d


@pytest.mark.parametrize("density", [0.002, 0.02, 0.2, 0.7])
def test_march_skipping_random_grids(dev, orc, density):
    rng = np.random.default_rng(int(density * 1000) + 11)
    R = 64
    mask = (rng.uniform(size=R ** 3) < density).astype(np.uint8)
    g = api.OccupancyGrid(R, Contraction.aabb(), dev=dev)
    og = orc.grid(R, O.Contraction.aabb())
    g.seed_mask(mask)
    og.seed_mask(mask)
    field = Field.box((0.1, 0.2, 0.0), (0.9, 0.7, 1.0), 30.0)
    o, d = _stress_rays(rng, 4000)
    for step in (0.003, 0.0117, 0.0371):
        cfg = MarchConfig(step, 1e-3, 1e-2)
        st = MarchStats()
        p = api.march(api.RayBatch.create(o, d, 0.0, 2.5, dev), g, field, cfg, stats=st)
        q = orc.march_field(o, d, 0.0, 2.5, og, ofield(field), ocfg(cfg), 4)
        same_packed(p, q)
        assert st.samples_emitted == q.samples_emitted


@pytest.mark.parametrize("R", [48, 64])
def test_march_bbox_clip_edges(dev, orc, R):
    """Rays are clipped to the occupied cells' bounding box (+ guard): occupied cells on
    the domain's faces and corners (the max face maps to cell R-1), a lone interior
    cell and a dense sub-box, crossed by axis-aligned rays, rays through the corners
    and rays starting on cell faces — identical samples and emitted counts."""
    rng = np.random.default_rng(R)
    field = Field.box((0.0, 0.0, 0.0), (1.0, 1.0, 1.0), 5.0)
    cases = []
    m = np.zeros((R, R, R), np.uint8)  # [z][y][x]
    m[R - 1, R - 1, R - 1] = 1
    m[0, 0, 0] = 1
    cases.append(m)
    m = np.zeros((R, R, R), np.uint8)
    m[:, :, R - 1] = rng.uniform(size=(R, R)) < 0.3  # x = R-1 face
    cases.append(m)
    m = np.zeros((R, R, R), np.uint8)
    m[R // 3, R // 2, R // 4] = 1
    cases.append(m)
    m = np.zeros((R, R, R), np.uint8)
    m[10:21, 5:17, 30:41] = rng.uniform(size=(11, 12, 11)) < 0.3
    cases.append(m)
    o, d = _stress_rays(rng, 3000)
    # rays aimed exactly at the corners / face centres from outside
    tgt = np.array([[0, 0, 0], [1, 1, 1], [1, 0.5, 0.5], [0.5, 1, 0.5], [1, 1, 0]], float)
    src = rng.uniform(-0.5, 1.5, (len(tgt) * 40, 3))
    dd = np.repeat(tgt, 40, 0) - src
    dd /= np.sqrt((dd * dd).sum(1))[:, None]
    o, d = np.concatenate([o, src]), np.concatenate([d, dd])
    for mask in cases:
        flat = mask.ravel()
        g = api.OccupancyGrid(R, Contraction.aabb(), dev=dev)
        og = orc.grid(R, O.Contraction.aabb())
        g.seed_mask(flat)
        og.seed_mask(flat)
        for step in (0.0041, 0.0173):
            cfg = MarchConfig(step, 1e-4, 1e-2)
            st = MarchStats()
            p = api.march(api.RayBatch.create(o, d, 0.0, 3.0, dev), g, field, cfg, stats=st)
            q = orc.march_field(o, d, 0.0, 3.0, og, ofield(field), ocfg(cfg), 4)
            same_packed(p, q)
            assert st.samples_emitted == q.samples_emitted


def test_march_grazing_sphere(dev, orc):
    """Rays tangent to the sphere at distance r +- tiny: the filtered fp32 density test
    must fall back to fp64 exactly where it matters."""
    field = Field.sphere(center=(0.5, 0.5, 0.5), radius=0.2, sigma=200.0)
    g, og = both_grids(dev, orc, 128, Contraction.aabb(), field, workload.grid_warmup_seeds(8, 5))
    rng = np.random.default_rng(5)
    n = 6000
    d = rng.normal(size=(n, 3))
    d /= np.sqrt((d * d).sum(1))[:, None]
    perp = rng.normal(size=(n, 3))
    perp -= (perp * d).sum(1)[:, None] * d
    perp /= np.sqrt((perp * perp).sum(1))[:, None]
    h = 0.2 + rng.choice([-1, 1], n) * 10.0 ** rng.uniform(-12, -3, n)
    o = 0.5 + perp * h[:, None] - d * 0.6
    for step in (5e-3, 1.6914558667664816e-3):
        cfg = MarchConfig(step, 1e-4, 1e-2)
        p = api.march(api.RayBatch.create(o, d, 0.2, 1.0, dev), g, field, cfg)
        same_packed(p, orc.march_field(o, d, 0.2, 1.0, og, ofield(field), ocfg(cfg), 4))


def test_march_float32_rays_match_widened_oracle(dev, orc):
    """The bench path: f32 rays on the device == the same rays widened to f64 on the CPU."""
    field = Field.sphere(**workload.SPHERE)
    g, og = both_grids(dev, orc, 128, Contraction.aabb(), field, workload.grid_warmup_seeds(16, 5))
    o, d = workload.orbit_rays(256, angle=1.3)
    o32, d32 = o.astype(np.float32), d.astype(np.float32)
    do_, dd_ = dev.upload(o32), dev.upload(d32)
    from paper_2210_04847_b200._lib import Rays, VMB_F32
    rays = Rays(do_.ptr, dd_.ptr, VMB_F32, 0, len(o), 0.2, 1.0)
    cfg = MarchConfig(5e-3, 1e-4, 1e-2)
    out = api.march_device(dev, g, rays, field, cfg, api.DevicePacked.allocate(dev, len(o), 16 * len(o)))
    same_packed(out.to_host(), orc.march_field(o32.astype(np.float64), d32.astype(np.float64), 0.2, 1.0,
                                               og, ofield(field), ocfg(cfg), 4))


@pytest.mark.parametrize("res,density", [(32, 0.01), (48, 0.002), (100, 0.0005), (128, 0.0), (40, 0.3)])
def test_distance_map_is_exact_capped_chebyshev(dev, res, density):
    """The marcher's acceleration structure: per cell the L-inf distance to the nearest
    occupied cell capped at 16 — exact (an over-estimate would skip candidates, an
    under-estimate only costs speed); resolutions not multiple of 32 included."""
    from scipy import ndimage
    rng = np.random.default_rng(res)
    occ = rng.random(res ** 3) < density
    if density > 0.2:  # clustered blobs too
        occ[: res * res * 3] = False
    g = api.OccupancyGrid(res, Contraction.aabb(), dev=dev)
    g.write(np.packbits(occ.astype(np.uint8), bitorder="little"))
    assert np.array_equal(g.bits(), occ.astype(np.uint8))
    dist, cap = g.distance_map()
    grid = occ.reshape(res, res, res)  # [z][y][x]
    if grid.any():
        want = ndimage.distance_transform_cdt(~grid, metric="chessboard")
    else:
        want = np.full(grid.shape, cap)
    want = np.minimum(want, cap).astype(np.uint8).ravel()
    assert np.array_equal(dist, want), np.argwhere(dist != want)[:5]
    # the ray clip box: the occupied cells' bounding box, exactly
    box = g.occupied_bbox()
    if grid.any():
        z, y, x = np.nonzero(grid)
        assert list(box) == [x.min(), y.min(), z.min(), x.max() + 1, y.max() + 1, z.max() + 1]
    else:
        assert all(box[a] >= box[3 + a] for a in range(3))


def test_render_backward_unaligned_buffers_match_aligned(dev, orc):
    """k_backward_hy stages groups with 16-byte bulk copies when every buffer is 16-byte
    aligned; buffers that are not (views into larger arrays at odd element offsets)
    take the per-element cp.async staging. Both agree bit for bit, and with the
    reference."""
    import ctypes as C
    from paper_2210_04847_b200._lib import VMB_F32, PackedView, check
    rng = np.random.default_rng(77)
    p, rgb, sig = _instance(rng, 3000, 40)
    n, s = p.n_rays, p.n_samples
    dc, do, dd = (rng.uniform(-1, 1, (n, 3)).astype(np.float32), rng.uniform(-1, 1, n).astype(np.float32),
                  rng.uniform(-1, 1, n).astype(np.float32))
    r32, s32 = rgb.astype(np.float32), sig.astype(np.float32)

    def run(shift):  # shift = elements of padding in front of every per-sample array
        pad = lambda a: np.concatenate([np.zeros(shift * (a.size // max(len(a), 1) if a.ndim > 1 else 1), a.dtype),
                                        a.reshape(-1)])  # noqa: E731
        off, cnt = dev.upload(p.offsets.astype(np.uint32)), dev.upload(p.counts.astype(np.uint32))
        ts, te = dev.upload(pad(p.t_starts)), dev.upload(pad(p.t_ends))
        dr, ds = dev.upload(pad(r32)), dev.upload(pad(s32))
        ups = [dev.upload(x.reshape(-1)) for x in (dc, do, dd)]
        gr, gs = dev.zeros((s + shift) * 3, np.float32), dev.zeros(s + shift, np.float32)
        v = PackedView(off.ptr, cnt.ptr, n, ts.ptr + 8 * shift, te.ptr + 8 * shift, s)
        check(dev.lib.vmb_render_backward(dev.h, C.byref(v), dr.ptr + 12 * shift, ds.ptr + 4 * shift,
                                          ups[0].ptr, ups[1].ptr, ups[2].ptr, gr.ptr + 12 * shift,
                                          gs.ptr + 4 * shift, VMB_F32))
        return gr.numpy((s + shift) * 3)[3 * shift:].reshape(s, 3), gs.numpy(s + shift)[shift:]

    a_rgb, a_sig = run(0)
    u_rgb, u_sig = run(1)
    assert np.array_equal(a_rgb, u_rgb) and np.array_equal(a_sig, u_sig)
    ref_r, ref_s = orc.render_backward(p, r32.astype(np.float64), s32.astype(np.float64), dc, do, dd)
    close(a_rgb, ref_r), close(a_sig, ref_s)

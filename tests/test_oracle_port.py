"""Pins the plain-C oracle restatement (oracle/vm_oracle.c) to the reference itself.

Every comparison here is bit-exact: both libraries run the same IEEE double
operations in the same order on the same inputs.
"""
import os
import tempfile

import numpy as np
import pytest

from oracle import Contraction, Field, MarchConfig, OracleError
from paper_2210_04847_b200 import workload

UNIT = Contraction.aabb()


def _rand_rays(rng, n, lo=0.0, hi=1.0, z=None):
    o = rng.uniform(lo, hi, (n, 3))
    if z is not None:
        o[:, 2] = z
    d = rng.normal(size=(n, 3))
    d /= np.sqrt((d * d).sum(1))[:, None]
    return o, d


def _same_packed(a, b):
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.samples_emitted == b.samples_emitted
    assert a.samples_kept == b.samples_kept


def _grids(ref, port, res, con, seeds, field, thr=1e-2, init=0.0, timestamps=(0.0,)):
    gr = ref.grid(res, con, thr, 0.0, init)
    gp = port.grid(res, con, thr, 0.0, init)
    for s in seeds:
        gr.update_field(field, 0.95, s, timestamps)
        gp.update_field(field, 0.95, s, timestamps)
    return gr, gp


def test_uniform_step_count(ref, port):
    rng = np.random.default_rng(0)
    for _ in range(2000):
        near = rng.uniform(0, 2)
        far = near + rng.choice([0.0, rng.uniform(0, 3)])
        step = rng.choice([1e-3, 5e-3, rng.uniform(1e-4, 0.5)])
        assert ref.uniform_step_count(near, far, step) == port.uniform_step_count(near, far, step)


def test_pack_and_validate(ref, port):
    rng = np.random.default_rng(1)
    for _ in range(50):
        counts = rng.integers(0, 12, rng.integers(0, 40)).astype(np.uint32)
        (o1, i1), (o2, i2) = ref.pack(counts), port.pack(counts)
        assert np.array_equal(o1, o2) and np.array_equal(i1, i2)
    with pytest.raises(OracleError) as e1:
        ref.pack(np.array([0x80000000, 0x80000001], np.uint32))
    with pytest.raises(OracleError) as e2:
        port.pack(np.array([0x80000000, 0x80000001], np.uint32))
    assert e1.value.msg == e2.value.msg == "pack: sample count exceeds 32-bit index range"
    # validate counterexamples (test_core_types.cpp:85-129 shapes)
    counts = np.array([2, 0, 3], np.uint32)
    off, idx = port.pack(counts)
    ts = np.array([0.1, 0.3, 0.0, 0.2, 0.5])
    te = np.array([0.2, 0.4, 0.1, 0.3, 0.6])
    cases = [
        (off, counts, ts, te, idx),
        (off[:2], counts, ts, te, idx),
        (np.array([0, 1, 2], np.uint32), counts, ts, te, idx),
        (off, counts, ts, np.where(np.arange(5) == 3, 0.2, te), idx),
        (off, counts, np.array([0.1, 0.3, 0.3, 0.2, 0.5]), te, idx),
        (off, counts, ts, np.array([0.2, 0.4, 0.1, 0.35, 0.6]), idx),
        (off, counts, ts, te, np.array([0, 0, 2, 1, 2], np.uint32)),
    ]
    for c in cases:
        assert ref.validate(*c) == port.validate(*c)


def test_contraction_functions(ref, port):
    rng = np.random.default_rng(2)
    sph = Contraction.sphere((0.5, 0.5, 0.5), 0.75)
    box = Contraction.aabb((-1, -2, 0.5), (2, 1, 1.5))
    x = rng.normal(scale=3.0, size=(5000, 3))
    g = rng.uniform(-0.1, 1.1, (5000, 3))
    for con in (sph, box, UNIT):
        assert np.array_equal(ref.contract(con, x), port.contract(con, x))
        a, va = ref.invert_grid_point(con, g)
        b, vb = port.invert_grid_point(con, g)
        assert np.array_equal(va, vb) and np.array_equal(a, b)
    with pytest.raises(OracleError) as e:
        port.contract(UNIT, [[np.nan, 0, 0]])
    assert e.value.msg == "non-finite coordinate"


@pytest.mark.parametrize("res,con_name", [(16, "unit"), (32, "box"), (24, "sphere")])
def test_grid_update_bits_and_cache(ref, port, res, con_name):
    con = {"unit": UNIT, "box": Contraction.aabb((-0.5, 0, 0), (1.5, 1, 2)),
           "sphere": Contraction.sphere((0.5, 0.5, 0.5), 0.5)}[con_name]
    field = Field.sphere(radius=0.3, sigma=60.0)
    seeds = [workload.mix_seed(99, i) for i in range(5)] + [None]
    gr, gp = _grids(ref, port, res, con, seeds, field)
    assert np.array_equal(gr.bits(), gp.bits())
    assert np.array_equal(gr.cache(), gp.cache())
    assert gr.info() == gp.info()
    pts = np.random.default_rng(3).uniform(-0.3, 1.3, (4000, 3))
    assert np.array_equal(gr.query(pts), gp.query(pts))


def test_grid_update_over_time_and_callback(ref, port):
    field = Field.sphere(center=(0.3, 0.5, 0.5), radius=0.15, sigma=80.0,
                         velocity=(-0.4, 0.0, 0.0))
    ts = [0.0, 0.5, 1.0]
    gr, gp = _grids(ref, port, 24, UNIT, [7, 8], field, timestamps=ts)
    assert np.array_equal(gr.bits(), gp.bits()) and np.array_equal(gr.cache(), gp.cache())

    def fn(p, t):
        return 30.0 * (np.sin(7 * p[:, 0] + t) > 0.3)

    gr2, gp2 = ref.grid(16, UNIT), port.grid(16, UNIT)
    gr2.update_callback(fn, 0.9, 11, (0.0, 2.0))
    gp2.update_callback(fn, 0.9, 11, (0.0, 2.0))
    assert np.array_equal(gr2.cache(), gp2.cache())
    # error naming the first offending cell (test_occupancy_grid.cpp:185-194)
    msgs = []
    for o in (ref, port):
        g = o.grid(4, UNIT)
        with pytest.raises(OracleError) as e:
            g.update_callback(lambda p, t: np.where(np.arange(len(p)) == 5, -2.0, 1.0), 0.95)
        msgs.append(e.value.msg)
    assert msgs[0] == msgs[1] == "occupancy grid: invalid density at cell (1,1,0)"


def test_seed_mask_and_ogrd_roundtrip(ref, port):
    rng = np.random.default_rng(4)
    mask = (rng.uniform(size=16 ** 3) < 0.4).astype(np.uint8)
    gr, gp = ref.grid(16, UNIT), port.grid(16, UNIT)
    gr.seed_mask(mask)
    gp.seed_mask(mask)
    assert np.array_equal(gr.bits(), gp.bits()) and np.array_equal(gr.cache(), gp.cache())
    with tempfile.TemporaryDirectory() as tmp:
        gs = ref.grid(16, Contraction.sphere((0.5, 0.5, 0.5), 0.75), 2e-2, 0.001)
        gs.update_field(Field.sphere(radius=0.4, sigma=60.0), 0.95, 1234)
        a, b = os.path.join(tmp, "a.ogrd"), os.path.join(tmp, "b.ogrd")
        gs.save(a)
        lp = port.grid_load(a)
        lp.save(b)
        assert open(a, "rb").read() == open(b, "rb").read()
        lr = ref.grid_load(b)
        assert np.array_equal(lr.bits(), lp.bits()) and np.array_equal(lr.cache(), lp.cache())


def _sphere_scene(ref, port, res=64, updates=4):
    field = Field.sphere(**workload.SPHERE)
    seeds = workload.grid_warmup_seeds(updates, 5)
    return field, _grids(ref, port, res, UNIT, seeds, field)


def test_march_field_matches_reference(ref, port):
    field, (gr, gp) = _sphere_scene(ref, port)
    o, d = workload.orbit_rays(48)
    for step, eps, thr in [(5e-3, 1e-4, 1e-2), (1.6914558667664816e-3, 1e-4, 1e-2),
                           (0.011, 0.0, 0.0), (5e-3, 0.5, 0.3)]:
        cfg = MarchConfig(step, eps, thr)
        a = ref.march_field(o, d, 0.2, 1.0, gr, field, cfg)
        b = port.march_field(o, d, 0.2, 1.0, gp, field, cfg)
        _same_packed(a, b)
    rng = np.random.default_rng(5)
    ro, rd = _rand_rays(rng, 300)
    cfg = MarchConfig(0.003, 1e-3, 0.0, max_samples_per_ray=17)
    _same_packed(ref.march_field(ro, rd, 0.0, 1.5, gr, field, cfg),
                 port.march_field(ro, rd, 0.0, 1.5, gp, field, cfg))


def test_march_growth_sphere_contraction(ref, port):
    con = Contraction.sphere((0.5, 0.5, 0.5), 0.5)
    field = Field.sphere(radius=0.3, sigma=40.0)
    gr, gp = _grids(ref, port, 32, con, [1, 2, 3], field)
    rng = np.random.default_rng(6)
    o = np.tile([[0.5, 0.5, 0.55]], (200, 1))
    _, d = _rand_rays(rng, 200)
    for growth in (1.0, 1.01, 1.05):
        cfg = MarchConfig(1.6914558667664816e-3 * 4, 1e-4, 1e-2, 2048, growth)
        _same_packed(ref.march_field(o, d, 0.01, 100.0, gr, field, cfg),
                     port.march_field(o, d, 0.01, 100.0, gp, field, cfg))


def test_march_callback_and_errors(ref, port):
    field, (gr, gp) = _sphere_scene(ref, port, res=32, updates=2)
    o, d = workload.orbit_rays(16)

    def sig(ts, te, idx):
        mid = 0.5 * (ts + te)
        return 50.0 * (0.5 + 0.5 * np.sin(20 * mid)) + idx * 0.0

    cfg = MarchConfig(0.01, 1e-3, 0.0)
    _same_packed(ref.march_callback(o, d, 0.2, 1.0, gr, sig, cfg),
                 port.march_callback(o, d, 0.2, 1.0, gp, sig, cfg))
    full_r, full_p = ref.grid(8, UNIT, 1e-2, 0.0, 1e6), port.grid(8, UNIT, 1e-2, 0.0, 1e6)
    ro, rd = np.array([[0.0, 0.5, 0.5]]), np.array([[1.0, 0.0, 0.0]])
    for bad, expect in [
        (lambda ts, te, idx: np.r_[np.ones(len(ts) - 1), np.nan],
         "marching: non-finite density at ray 0 sample 7"),
        (lambda ts, te, idx: np.ones(len(ts) + 1), "marching: sigma_fn returned 9 values for 8 samples"),
        (lambda ts, te, idx: np.r_[-np.ones(1), np.ones(len(ts) - 1)],
         "marching: negative density at ray 0 sample 0"),
    ]:
        msgs = []
        for o_, g in ((ref, full_r), (port, full_p)):
            with pytest.raises(OracleError) as e:
                o_.march_callback(ro, rd, 0.2, 1.0, g, bad, MarchConfig(0.1))
            msgs.append(e.value.msg)
        assert msgs == [expect, expect]


def test_march_uniform(ref, port):
    rng = np.random.default_rng(7)
    o, d = _rand_rays(rng, 50)
    for near, far, step in [(0.2, 1.0, 0.1), (0.2, 0.25, 0.1), (0.0, 3.0, 0.0137)]:
        cfg = MarchConfig(step)
        _same_packed(ref.march_uniform(o, d, near, far, cfg), port.march_uniform(o, d, near, far, cfg))


def _random_instance(rng, max_rays=40, max_per_ray=20):
    """random_instance (test_rendering.cpp:40-64) shape, numpy-seeded."""
    counts = rng.integers(0, max_per_ray + 1, rng.integers(0, max_rays + 1)).astype(np.uint32)
    offsets = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint32) if len(counts) else np.zeros(0, np.uint32)
    ts, te = [], []
    for c in counts:
        t = rng.uniform(0, 0.5)
        for _ in range(c):
            w = rng.uniform(0.01, 0.2)
            ts.append(t)
            te.append(t + w)
            t += w
    from oracle import Packed
    idx = np.repeat(np.arange(len(counts), dtype=np.uint32), counts)
    p = Packed(offsets, counts, np.array(ts, float), np.array(te, float), idx)
    s = p.n_samples
    return p, rng.uniform(0, 1, (s, 3)), rng.uniform(0, 8, s)


def test_rendering_matches_reference(ref, port):
    rng = np.random.default_rng(8)
    for _ in range(30):
        p, rgb, sig = _random_instance(rng)
        n = p.n_rays
        dc, do, dd = rng.uniform(-1, 1, (n, 3)), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        assert np.array_equal(ref.transmittance(p, sig), port.transmittance(p, sig))
        for a, b in zip(ref.render_forward(p, rgb, sig), port.render_forward(p, rgb, sig)):
            assert np.array_equal(a, b)
        for a, b in zip(ref.render_backward(p, rgb, sig, dc, do, dd),
                        port.render_backward(p, rgb, sig, dc, do, dd)):
            assert np.array_equal(a, b)
        vals = rng.uniform(-2, 2, (p.n_samples, 3))
        assert np.array_equal(ref.render_attribute(p, sig, vals, 3),
                              port.render_attribute(p, sig, vals, 3))


def test_shade_and_train_step(ref, port):
    field, (gr, gp) = _sphere_scene(ref, port, res=32, updates=3)
    o, d = workload.orbit_rays(32)
    cfg = MarchConfig(5e-3)
    p = ref.march_field(o, d, 0.2, 1.0, gr, field, cfg)
    for f in (field, Field.checker(0.1, 3.0, (0.9, 0.1, 0.2), (0.1, 0.8, 0.3)),
              Field.box((0.3, 0.3, 0.3), (0.7, 0.6, 0.8), 5.0, (0.2, 0.3, 0.4))):
        a, b = ref.shade(o, d, p, f), port.shade(o, d, p, f)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    dc, do, dd = workload.upstream_grads(len(o))
    _, n1, c1 = ref.train_step(o, d, 0.2, 1.0, gr, field, cfg, dc, do, dd, 2)
    _, n2, c2 = port.train_step(o, d, 0.2, 1.0, gp, field, cfg, dc, do, dd, 1)
    assert n1 == n2 and c1 == c2

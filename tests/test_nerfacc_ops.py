"""NerfAcc's standalone operators (render_weight_from_density / _from_alpha,
render_transmittance_from_alpha, accumulate_along_rays — forward and backward —
and ray_aabb_intersect).

The reference has no such functions: it composites only inside render_forward /
render_backward (rendering.cpp:47-58, 67-112) and transmittance (:19-33). The
oracle port's sequential restatement (oracle/vm_oracle.c, vmo_weight_from_density
...) is therefore pinned against the reference by DECOMPOSITION:

  * accumulate(weights, rgb) == render_forward's color, accumulate(weights) ==
    opacity, accumulate(weights, mid) == depth — bit for bit (same products, same
    summation order);
  * the density backward with grad_weights = render_backward's per-sample value
    v = dot(d_color, rgb) + d_opacity + d_depth mid is render_backward's d_sigma,
    bit for bit (rendering.cpp:99-108's suffix form);
  * transmittance from alpha == transmittance() within 1e-12 (the reference
    multiplies exp(-sigma delta), rendering.cpp:29, the operator 1 - alpha);
  * every backward against central finite differences (test_rendering.cpp:253-293);
  * ray_aabb_intersect against OccupancyGrid::query's domain reject
    (occupancy_grid.cpp:69) on a fully occupied grid.

The CUDA kernels (csrc/ops.cu, warp-shuffle segmented scans) are compared with the
port under -m gpu (a few ulps: the scans reassociate products and sums).
"""
import numpy as np
import pytest

from oracle import Oracle, available
from oracle import oracle as O
from oracle.oracle import NerfaccOracle

needs_ref = pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def nf():
    return NerfaccOracle()


def instance(rng, n_rays, max_per_ray, contiguous=True, zero_frac=0.2, sigma_hi=8.0):
    counts = rng.integers(0, max_per_ray + 1, n_rays).astype(np.uint32)
    counts[rng.uniform(size=n_rays) < zero_frac] = 0
    offsets = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint32)
    s = int(counts.sum())
    ts, te = np.empty(s), np.empty(s)
    for r in range(n_rays):
        b, c = offsets[r], counts[r]
        w = rng.uniform(0.01, 0.2, c)
        t0 = rng.uniform(0, 0.5) + np.concatenate([[0], np.cumsum(w)[:-1]])
        ts[b:b + c], te[b:b + c] = t0, t0 + w
    if not contiguous:  # store the rays in reverse order: offsets descend
        new_off, at = np.zeros(n_rays, np.uint32), 0
        ts2, te2 = np.empty(s), np.empty(s)
        for r in range(n_rays)[::-1]:
            b, c = offsets[r], counts[r]
            ts2[at:at + c], te2[at:at + c] = ts[b:b + c], te[b:b + c]
            new_off[r] = at
            at += c
        offsets, ts, te = new_off, ts2, te2
    p = O.Packed(offsets, counts, ts, te, np.zeros(s, np.uint32))
    return p, rng.uniform(0, sigma_hi, s)


def per_sample_value(p, rgb, dc, do, dd):
    """render_backward's value (rendering.cpp:101-102), same operation order."""
    ray = np.repeat(np.arange(p.n_rays), p.counts)
    order = np.concatenate([np.arange(o, o + c) for o, c in zip(p.offsets, p.counts)]) if p.n_samples else []
    v = np.zeros(p.n_samples)
    mid = 0.5 * (p.t_starts + p.t_ends)
    s = np.asarray(order, dtype=np.int64)
    dot = (dc[ray, 0] * rgb[s, 0] + dc[ray, 1] * rgb[s, 1]) + dc[ray, 2] * rgb[s, 2]
    v[s] = (dot + do[ray]) + dd[ray] * mid[s]
    return v


@needs_ref
def test_forward_decomposes_render_forward_bit_exact(nf):
    orc = Oracle("ref")
    rng = np.random.default_rng(1)
    p, sig = instance(rng, 300, 40)
    rgb = rng.uniform(0, 1, (p.n_samples, 3))
    col, op, dep = orc.render_forward(p, rgb, sig)
    w, t, a = nf.weight_from_density(p, sig)
    assert np.array_equal(nf.accumulate_along_rays(p, w)[:, 0], op)
    assert np.array_equal(nf.accumulate_along_rays(p, w, rgb, 3), col)
    mid = 0.5 * (p.t_starts + p.t_ends)
    assert np.array_equal(nf.accumulate_along_rays(p, w, mid)[:, 0], dep)
    # render_attribute is the same weighted reduce (rendering.cpp:114-134)
    assert np.array_equal(nf.accumulate_along_rays(p, w, rgb, 3).ravel(), orc.render_attribute(p, sig, rgb, 3))
    # transmittance(): exp products instead of (1 - alpha) products
    tr = orc.transmittance(p, sig)
    assert np.allclose(t, tr, rtol=1e-12, atol=1e-15)
    wa, ta = nf.weight_from_alpha(p, a)
    assert np.array_equal(wa, w) and np.array_equal(ta, t)


@needs_ref
def test_density_backward_is_render_backward_bit_exact(nf):
    orc = Oracle("ref")
    rng = np.random.default_rng(2)
    p, sig = instance(rng, 300, 40)
    rgb = rng.uniform(0, 1, (p.n_samples, 3))
    n = p.n_rays
    dc, do, dd = rng.uniform(-1, 1, (n, 3)), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    _, ref_sig = orc.render_backward(p, rgb, sig, dc, do, dd)
    v = per_sample_value(p, rgb, dc, do, dd)
    got = nf.weight_from_density_backward(p, sig, v)
    assert np.array_equal(got, ref_sig)


def _fd(f, x, i, h):
    xp, xm = x.copy(), x.copy()
    xp[i] += h
    xm[i] -= h
    return (f(xp) - f(xm)) / (2 * h)


def test_backward_finite_differences(nf):
    """test_rendering.cpp:253-293 pattern: a scalar loss L = sum g * output."""
    rng = np.random.default_rng(3)
    for inst in range(12):
        p, sig = instance(rng, 4, 6, zero_frac=0.0, sigma_hi=5.0)
        s = p.n_samples
        gw, gt, ga = rng.uniform(-1, 1, s), rng.uniform(-1, 1, s), rng.uniform(-1, 1, s)

        def loss_d(x):
            w, t, a = nf.weight_from_density(p, x)
            return float(np.dot(gw, w) + np.dot(gt, t) + np.dot(ga, a))

        g = nf.weight_from_density_backward(p, sig, gw, gt, ga)
        alphas = rng.uniform(0.0, 0.9, s)

        def loss_a(x):
            w, t = nf.weight_from_alpha(p, x)
            return float(np.dot(gw, w) + np.dot(gt, t))

        ga_ = nf.weight_from_alpha_backward(p, alphas, gw, gt)
        gt_only = nf.weight_from_alpha_backward(p, alphas, None, gt)
        for i in range(s):
            fd = _fd(loss_d, sig, i, 1e-6)
            assert abs(fd - g[i]) <= 1e-5 * max(1.0, abs(fd)), (inst, i, fd, g[i])
            fd = _fd(loss_a, alphas, i, 1e-6)
            assert abs(fd - ga_[i]) <= 1e-5 * max(1.0, abs(fd)), (inst, i, fd, ga_[i])
            fd = _fd(lambda x: float(np.dot(gt, nf.weight_from_alpha(p, x)[1])), alphas, i, 1e-6)
            assert abs(fd - gt_only[i]) <= 1e-5 * max(1.0, abs(fd))
        vals = rng.uniform(-1, 1, (s, 2))
        go = rng.uniform(-1, 1, (p.n_rays, 2))
        w = rng.uniform(0, 1, s)
        gw2, gv2 = nf.accumulate_along_rays_backward(p, w, vals, 2, go)
        for i in range(s):
            fd = _fd(lambda x: float(np.sum(go * nf.accumulate_along_rays(p, x, vals, 2))), w, i, 1e-6)
            assert abs(fd - gw2[i]) <= 1e-6 * max(1.0, abs(fd))
        ray = np.repeat(np.arange(p.n_rays), p.counts)
        assert np.allclose(gv2, w[:, None] * go[ray])


def test_density_backward_chain_rule_matches_alpha_backward(nf):
    """dL/dsigma = delta (1 - alpha) dL/dalpha: the suffix form (density) and the
    division-free reverse recurrence (alpha) agree to rounding."""
    rng = np.random.default_rng(4)
    p, sig = instance(rng, 200, 30)
    s = p.n_samples
    gw, gt = rng.uniform(-1, 1, s), rng.uniform(-1, 1, s)
    _, _, a = nf.weight_from_density(p, sig)
    gd = nf.weight_from_density_backward(p, sig, gw, gt)
    gal = nf.weight_from_alpha_backward(p, a, gw, gt)
    delta = p.t_ends - p.t_starts
    assert np.allclose(gd, delta * (1.0 - a) * gal, rtol=1e-9, atol=1e-13)


@needs_ref
def test_ray_aabb_matches_grid_domain_reject(nf):
    """A fully occupied AABB grid accepts exactly the points inside [lo, hi]: the
    points o + t d with t strictly inside (t_min, t_max) are accepted by the
    reference's query, the others rejected (away from a 1e-9 band at the faces)."""
    orc = Oracle("ref")
    lo, hi = np.array([-0.3, 0.1, 0.2]), np.array([0.9, 1.4, 0.8])
    g = orc.grid(8, O.Contraction.aabb(tuple(lo), tuple(hi)))
    g.seed_mask(np.ones(8 ** 3, np.uint8))
    rng = np.random.default_rng(5)
    o = rng.uniform(-1.5, 2.0, (400, 3))
    d = rng.normal(size=(400, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d[:20, 0] = 0.0  # axis-parallel rays
    d[:20] /= np.linalg.norm(d[:20], axis=1, keepdims=True)
    tmin, tmax, hit = nf.ray_aabb_intersect(o, d, np.concatenate([lo, hi])[None])
    ts = np.linspace(-4, 4, 801)
    for r in range(len(o)):
        pts = o[r] + ts[:, None] * d[r]
        inside = g.query(pts)
        if not hit[r, 0]:
            assert not inside.any()
            continue
        band = (np.abs(ts - tmin[r, 0]) < 1e-9) | (np.abs(ts - tmax[r, 0]) < 1e-9)
        want = (ts > tmin[r, 0]) & (ts < tmax[r, 0])
        assert np.array_equal(inside[~band], want[~band]), r
    # near/far clamp and the miss value
    t2, u2, h2 = nf.ray_aabb_intersect(o, d, np.concatenate([lo, hi])[None], 0.0, 1.0, -1.0)
    assert np.all(t2[h2] >= 0.0) and np.all(u2[h2] <= 1.0) and np.all(t2[~h2] == -1.0)


# ------------------------------------------------------------------ device vs port
def _close(a, b, rtol, atol):
    a, b = np.asarray(a, float), np.asarray(b, float)
    assert a.shape == b.shape
    bad = np.abs(a - b) > np.maximum(rtol * np.maximum(np.abs(a), np.abs(b)), atol)
    assert not bad.any(), f"{bad.sum()} of {bad.size} differ, worst {np.abs(a - b).max()}"


@pytest.mark.gpu
@pytest.mark.parametrize("n_rays,max_per_ray,contiguous", [(3000, 12, True), (257, 300, True), (200, 40, False),
                                                           (40, 3000, True), (5, 5000, False)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_device_ops_match_port(nf, n_rays, max_per_ray, contiguous, dtype):
    from paper_2210_04847_b200 import api
    dev = api.Device(0)
    rng = np.random.default_rng(n_rays + max_per_ray)
    p, sig = instance(rng, n_rays, max_per_ray, contiguous, sigma_hi=2.0)
    s = p.n_samples
    ap = api.PackedSamples(p.offsets, p.counts, p.t_starts, p.t_ends, p.ray_indices)
    r = lambda x: np.asarray(x, dtype).astype(np.float64)  # noqa: E731
    rtol, atol = (1e-10, 1e-13) if dtype == np.float64 else (1e-5, 1e-7)
    sig = r(sig)
    gw, gt, ga = (r(rng.uniform(-1, 1, s)) for _ in range(3))
    w, t, a = api.render_weight_from_density(ap, sig, dev=dev, dtype=dtype)
    ow, ot, oa = nf.weight_from_density(p, sig)
    for x, y in ((w, ow), (t, ot), (a, oa)):
        _close(x, y, rtol, atol)
    _close(api.render_weight_from_density_backward(ap, sig, gw, gt, ga, dev=dev, dtype=dtype),
           nf.weight_from_density_backward(p, sig, gw, gt, ga), rtol, atol * 10)
    _close(api.render_weight_from_density_backward(ap, sig, gw, dev=dev, dtype=dtype),
           nf.weight_from_density_backward(p, sig, gw), rtol, atol * 10)
    al = r(rng.uniform(0, 0.3, s))
    w2, t2 = api.render_weight_from_alpha(ap, al, dev=dev, dtype=dtype)
    ow2, ot2 = nf.weight_from_alpha(p, al)
    _close(w2, ow2, rtol, atol)
    _close(t2, ot2, rtol, atol)
    _close(api.render_transmittance_from_alpha(ap, al, dev=dev, dtype=dtype), ot2, rtol, atol)
    _close(api.render_weight_from_alpha_backward(ap, al, gw, gt, dev=dev, dtype=dtype),
           nf.weight_from_alpha_backward(p, al, gw, gt), rtol, atol * 10)
    _close(api.render_transmittance_from_alpha_backward(ap, al, gt, dev=dev, dtype=dtype),
           nf.weight_from_alpha_backward(p, al, None, gt), rtol, atol * 10)
    vals = r(rng.uniform(-1, 1, (s, 3)))
    _close(api.accumulate_along_rays(ap, ow, vals, 3, dev=dev, dtype=dtype),
           nf.accumulate_along_rays(p, r(ow), vals, 3), rtol, atol)
    _close(api.accumulate_along_rays(ap, ow, None, 1, dev=dev, dtype=dtype),
           nf.accumulate_along_rays(p, r(ow)), rtol, atol)
    go = r(rng.uniform(-1, 1, (p.n_rays, 3)))
    g1, g2 = api.accumulate_along_rays_backward(ap, ow, vals, 3, go, dev=dev, dtype=dtype)
    o1, o2 = nf.accumulate_along_rays_backward(p, r(ow), vals, 3, go)
    _close(g1, o1, rtol, atol)
    _close(g2, o2, rtol, atol)


@pytest.mark.gpu
def test_device_ray_aabb_bit_exact(nf):
    from paper_2210_04847_b200 import api
    dev = api.Device(0)
    rng = np.random.default_rng(6)
    o = rng.uniform(-2, 2, (5000, 3))
    d = rng.normal(size=(5000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d[:100, 1] = 0.0
    boxes = np.concatenate([rng.uniform(-1, 0, (3, 3)), rng.uniform(0.1, 1.5, (3, 3))], axis=1)
    for near, far, miss in ((-np.inf, np.inf, np.inf), (0.0, 2.5, -1.0)):
        got = api.ray_aabb_intersect(o, d, boxes, near, far, miss, dev=dev)
        want = nf.ray_aabb_intersect(o, d, boxes, near, far, miss)
        for x, y in zip(got, want):
            assert np.array_equal(x, y)

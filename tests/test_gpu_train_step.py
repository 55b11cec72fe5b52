"""The fused training step (vmb_march_render_backward_field_async): march +
shading + render_forward + render_backward in one call, the backward computed by
the expansion from the samples it has just produced.

Against the two-call path (vmb_march_render_field_async -> vmb_render_backward) on
the same inputs: packing, rgb/sigma and color/opacity/depth bit for bit (the same
kernels produce them); d_rgb / d_sigma within the rendering tolerance (the fused
backward's T products and suffix sums are warp scans, the two-call backward's are
the reference's sequential loops) — and both against the reference's
render_backward. Covers the constant-density table (SolidSphere), a per-sample
field (Checker), the stored voxel field, f64 attributes, and rays with more than
the expansion's 32 kept samples (their chunks fall back to k_backward_long).
"""
import numpy as np
import pytest

from oracle import Oracle, available
from oracle import oracle as O
from paper_2210_04847_b200 import api, workload
from paper_2210_04847_b200._lib import VMB_F32, VMB_F64, Contraction, Field, MarchConfig, Rays, check

pytestmark = pytest.mark.gpu
RTOL, ATOL = 1e-5, 1e-8


def close(a, b, what, rtol=RTOL, atol=ATOL):
    a, b = np.asarray(a, float), np.asarray(b, float)
    assert a.shape == b.shape, what
    bad = np.abs(a - b) > np.maximum(rtol * np.maximum(np.abs(a), np.abs(b)), atol)
    assert not bad.any(), f"{what}: {bad.sum()} mismatches, worst {np.abs(a - b).max()}"


@pytest.fixture(scope="module")
def dev():
    return api.Device(0)


def ofield(f):
    o = O.Field()
    for name, _ in Field._fields_:
        setattr(o, name, getattr(f, name))
    return o


def _voxel(dev):
    res = 48
    vf = api.VoxelField(res, (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), dev=dev)
    g = np.arange(res) / (res - 1)
    x, y, z = np.meshgrid(g, g, g, indexing="ij")
    inside = ((x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2) <= 0.25 ** 2
    dens = np.where(inside, 60.0, -20.0).transpose(2, 1, 0).ravel()
    col = np.random.default_rng(0).normal(size=(res ** 3, 3))
    vf.set_params(dens, col)
    return vf


def _step(dev, grid, field, cfg, o, d, ups, dtype, fused):
    n = len(o)
    dt = np.float32 if dtype == VMB_F32 else np.float64
    do_, dd_ = dev.upload(o.astype(np.float32)), dev.upload(d.astype(np.float32))
    rays = Rays(do_.ptr, dd_.ptr, VMB_F32, 0, n, 0.2, 1.0)
    p = api.DevicePacked.allocate(dev, n, 400 * n)
    cap = p.capacity
    rgb, sig = dev.empty(3 * cap, dt), dev.empty(cap, dt)
    outs = [dev.empty(3 * n, dt), dev.empty(n, dt), dev.empty(n, dt)]
    du = [dev.upload(x.astype(dt)) for x in ups]
    gr, gs = dev.zeros(3 * cap, dt), dev.zeros(cap, dt)
    n_dev = dev.zeros(1, np.uint64)
    if fused:
        api.march_render_backward_device(dev, grid, rays, field, cfg, p, rgb, sig, *outs, *du, gr, gs, n_dev)
    else:
        smp = p.samples_struct()
        import ctypes as C
        check(dev.lib.vmb_march_render_field_async(dev.h, grid.h, C.byref(rays), C.byref(field), C.byref(cfg),
                                                   C.byref(smp), rgb.ptr, sig.ptr, outs[0].ptr, outs[1].ptr,
                                                   outs[2].ptr, dtype, 0.0, n_dev.ptr))
        p.n_samples = cap
        api.render_backward_device(dev, p, rgb, sig, *du, gr, gs)
    dev.sync()
    check(dev.lib.vmb_march_check(dev.h))
    s = int(n_dev.numpy()[0])
    assert s <= cap
    p.n_samples = s
    h = p.to_host()
    return dict(packed=h, rgb=rgb.numpy(3 * s).reshape(-1, 3), sig=sig.numpy(s),
                outs=[outs[0].numpy(3 * n).reshape(-1, 3), outs[1].numpy(n), outs[2].numpy(n)],
                gr=gr.numpy(3 * s).reshape(-1, 3), gs=gs.numpy(s))


CASES = {
    "sphere": (lambda dev: (Field.sphere(**workload.SPHERE), None), MarchConfig(5e-3, 1e-4, 1e-2)),
    "sphere_fine": (lambda dev: (Field.sphere(**workload.SPHERE), None), MarchConfig(1.6914558667664816e-3)),
    "long_rays": (lambda dev: (Field.sphere(radius=0.3, sigma=6.0), None), MarchConfig(2e-3, 1e-4, 1e-3)),
    "checker": (lambda dev: (Field.checker(period=0.0625, sigma=80.0, rgb_a=(0.9, 0.2, 0.1),
                                           rgb_b=(0.1, 0.3, 0.8)), None), MarchConfig(5e-3, 1e-4, 1e-2)),
    "voxel": (lambda dev: (lambda vf: (vf.field, vf))(_voxel(dev)), MarchConfig(5e-3, 1e-4, 1e-2)),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("dtype", [VMB_F32, VMB_F64])
def test_fused_train_step_matches_two_calls_and_reference(dev, case, dtype):
    make, cfg = CASES[case]
    field, keep = make(dev)
    grid = api.OccupancyGrid(64, Contraction.aabb(), dev=dev)
    for s in workload.grid_warmup_seeds(6, 5):
        grid.update_field(field, 0.95, s)
    o, d = workload.orbit_rays(160)
    ups = workload.upstream_grads(len(o), 21)
    a = _step(dev, grid, field, cfg, o, d, ups, dtype, fused=True)
    b = _step(dev, grid, field, cfg, o, d, ups, dtype, fused=False)
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(a["packed"], k), getattr(b["packed"], k)), k
    assert np.array_equal(a["rgb"], b["rgb"]) and np.array_equal(a["sig"], b["sig"])
    for x, y in zip(a["outs"], b["outs"]):
        assert np.array_equal(x, y)
    if case == "long_rays":
        assert int(a["packed"].counts.max()) > 32  # chunks that take the listed fallback
    tol = (1e-5, 1e-8) if dtype == VMB_F32 else (1e-10, 1e-13)
    close(a["gr"], b["gr"], "d_rgb", *tol)
    close(a["gs"], b["gs"], "d_sigma", *tol)
    orc = Oracle("ref") if available("ref") else Oracle("port")
    ref = O.Packed(a["packed"].offsets, a["packed"].counts, a["packed"].t_starts, a["packed"].t_ends,
                   a["packed"].ray_indices)
    dt = np.float32 if dtype == VMB_F32 else np.float64
    rg, rs = orc.render_backward(ref, a["rgb"].astype(np.float64), a["sig"].astype(np.float64),
                                 *[x.astype(dt).astype(np.float64) for x in ups])
    close(a["gr"], rg, "d_rgb vs reference")
    close(a["gs"], rs, "d_sigma vs reference")
    del keep

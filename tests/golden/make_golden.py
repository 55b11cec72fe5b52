"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the dev container (needs oracle/_ref/libvoxmarch_ref.so, built from
/root/reference by `make -C oracle`):

    python tests/golden/make_golden.py

Fixtures (numpy .npz, compressed):
  c1.npz   BASELINE config 1: 64x64 orbit rays, 128^3 grid warmed by 16 jittered
           updates (Rng(5) seeds), step 5e-3 — grid bits, packed samples, MarchStats,
           shaded attributes, render_forward outputs and render_backward gradients
           for upstream gradients from workload.upstream_grads(seed=113).
  growth.npz  sphere contraction + step growth 1.01 (config-3 stand-in, 24^2 rays, 64^3).
  render.npz  60 random packed instances (test_rendering.cpp:40-64 shape) with
           transmittance / forward / backward / attribute outputs.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import Contraction, Field, MarchConfig, Oracle  # noqa: E402
from paper_2210_04847_b200 import workload  # noqa: E402


def config1(ref):
    field = Field.sphere(**workload.SPHERE)
    g = ref.grid(128, Contraction.aabb())
    for s in workload.grid_warmup_seeds(16, 5):
        g.update_field(field, 0.95, s)
    o, d = workload.orbit_rays(64)
    cfg = MarchConfig(5e-3, 1e-4, 1e-2)
    p = ref.march_field(o, d, 0.2, 1.0, g, field, cfg)
    rgb, sig = ref.shade(o, d, p, field)
    color, op, dep = ref.render_forward(p, rgb, sig)
    dc, do, dd = workload.upstream_grads(len(o), seed=113)
    d_rgb, d_sig = ref.render_backward(p, rgb, sig, dc, do, dd)
    return dict(bits=np.packbits(g.bits(), bitorder="little"), cache=g.cache().astype(np.float32),
                offsets=p.offsets, counts=p.counts, t_starts=p.t_starts, t_ends=p.t_ends,
                ray_indices=p.ray_indices, emitted=p.samples_emitted, kept=p.samples_kept,
                rgbs=rgb, sigmas=sig, color=color, opacity=op, depth=dep, d_color=dc,
                d_opacity=do, d_depth=dd, d_rgbs=d_rgb, d_sigmas=d_sig,
                occupied_fraction=g.info()["occupied_fraction"])


def growth(ref):
    con = Contraction.sphere((0.5, 0.5, 0.5), 0.5)
    field = Field.sphere(radius=0.3, sigma=40.0)
    g = ref.grid(64, con)
    for s in (1, 2, 3):
        g.update_field(field, 0.95, s)
    o, d = workload.orbit_rays(24, near=0.01, far=100.0)
    o[:] = [0.5, 0.5, 0.55]
    cfg = MarchConfig(1.6914558667664816e-3, 1e-4, 1e-2, 2048, 1.01)
    p = ref.march_field(o, d, 0.01, 100.0, g, field, cfg)
    return dict(bits=np.packbits(g.bits(), bitorder="little"), origins=o, dirs=d,
                offsets=p.offsets, counts=p.counts, t_starts=p.t_starts, t_ends=p.t_ends,
                ray_indices=p.ray_indices, emitted=p.samples_emitted, kept=p.samples_kept)


def render(ref):
    rng = np.random.default_rng(2024)
    out = {}
    for i in range(60):
        counts = rng.integers(0, 17, rng.integers(0, 9)).astype(np.uint32)
        offsets = (np.concatenate([[0], np.cumsum(counts)[:-1]]) if len(counts) else np.zeros(0)).astype(np.uint32)
        ts, te = [], []
        for c in counts:
            t = rng.uniform(0, 0.5)
            for _ in range(c):
                w = rng.uniform(0.01, 0.2)
                ts.append(t)
                te.append(t + w)
                t += w
        from oracle import Packed
        p = Packed(offsets, counts, np.array(ts, float), np.array(te, float),
                   np.repeat(np.arange(len(counts), dtype=np.uint32), counts))
        s, n = p.n_samples, p.n_rays
        rgb, sig = rng.uniform(0, 1, (s, 3)), rng.uniform(0, 8, s)
        dc, do, dd = rng.uniform(-1, 1, (n, 3)), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        vals = rng.uniform(-2, 2, (s, 2))
        color, op, dep = ref.render_forward(p, rgb, sig)
        d_rgb, d_sig = ref.render_backward(p, rgb, sig, dc, do, dd)
        for k, v in dict(offsets=offsets, counts=counts, t_starts=p.t_starts, t_ends=p.t_ends,
                         rgbs=rgb, sigmas=sig, d_color=dc, d_opacity=do, d_depth=dd,
                         values=vals, trans=ref.transmittance(p, sig), color=color, opacity=op,
                         depth=dep, d_rgbs=d_rgb, d_sigmas=d_sig,
                         attr=ref.render_attribute(p, sig, vals, 2)).items():
            out[f"{i}_{k}"] = v
    return out


def main():
    ref = Oracle("ref")
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **config1(ref))
    np.savez_compressed(os.path.join(HERE, "growth.npz"), **growth(ref))
    np.savez_compressed(os.path.join(HERE, "render.npz"), **render(ref))
    for f in ("c1.npz", "growth.npz", "render.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
